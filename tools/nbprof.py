"""Experiment: per-CTA phase timestamps of k_nonbonded (library built with -DNB_EXP_PROF)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["REAX_SERIAL"] = "1"
import gen
import paper_1706_07772_b200 as rx
lib = rx.load_library()
s = gen.make_config(1)
p = gen.make_params()
dev = torch.device("cuda:0")
ctx = rx.Reax(len(s.pos), s.box, p, gen.CUTOFFS, device=dev)
pos = torch.from_numpy(s.pos).to(dev); typ = torch.from_numpy(s.type).to(dev); q = torch.from_numpy(s.q).to(dev)
for _ in range(3):
    ctx.step(pos, typ, q)
torch.cuda.synchronize()
nb = 686
buf = (ctypes.c_ulonglong * (16 * 8192))()
lib.reax_exp_nbprof(buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 16)[:nb].astype(np.int64)
t0 = a[:, 0].min()
start, setup, end, sm = a[:, 0] - t0, a[:, 1] - t0, a[:, 2] - t0, a[:, 3]
wend = a[:, 4:12] - t0
print("kernel span us", (end.max() - start.min()) / 1e3)
print("per CTA: setup us mean %.2f, compute (setup->last warp) mean %.2f, warp spread (last-first) mean %.2f, flush (last warp->end) mean %.2f, total mean %.2f" % (
    (setup - start).mean() / 1e3, (wend.max(1) - setup).mean() / 1e3, (wend.max(1) - wend.min(1)).mean() / 1e3,
    (end - wend.max(1)).mean() / 1e3, (end - start).mean() / 1e3))
for smid in [0, 70]:
    idx = np.where(sm == smid)[0]
    idx = idx[np.argsort(start[idx])]
    print("SM", smid, [(int(start[i] / 1e3), int((setup[i] - start[i]) / 1e3 * 10) / 10, int((wend[i].max() - setup[i]) / 1e2) / 10, int((end[i] - wend[i].max()) / 1e2) / 10) for i in idx])

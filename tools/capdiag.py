"""Print the capacities a sync step regrows to (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1706_07772_b200 as rx
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
s = gen.make_config(k); p = gen.make_params(); dev = torch.device("cuda:0")
ctx = rx.Reax(len(s.pos), s.box, p, gen.CUTOFFS, device=dev)
c0 = (ctx.cap.row_cap, ctx.cap.cand_cap, ctx.cap.bond_cap, ctx.cap.window_cap)
F, E = ctx.step(*(torch.from_numpy(x).to(dev) for x in (s.pos, s.type, s.q)))
torch.cuda.synchronize()
print("cap before", c0, "after", (ctx.cap.row_cap, ctx.cap.cand_cap, ctx.cap.bond_cap, ctx.cap.window_cap))

# usage: bash tools/gpu_variants.sh lib1.so lib2.so ...  -- quick parity (c0/c1) + serial and forked bench per library
set -x
mkdir -p gpurun_out
for L in "$@"; do
  T=$(basename $L .so)
  REAX_LIBRARY=$PWD/$L timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:cacheprovider -k "c0_full or c1_full or deterministic or graph" > gpurun_out/var_$T.test 2>&1; tail -1 gpurun_out/var_$T.test
  REAX_LIBRARY=$PWD/$L REAX_SERIAL=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/var_${T}_serial.json 2>/dev/null
  REAX_LIBRARY=$PWD/$L timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/var_${T}.json 2>/dev/null
  python - "$T" <<'PY'
import json, sys
t = sys.argv[1]
for suf in ("_serial", ""):
    d = json.load(open(f"gpurun_out/var_{t}{suf}.json"))
    print(t + suf, "ms/step %.4f" % d["ms_per_step"], {k: round(v * 1000, 1) for k, v in d["kernel_ms_per_step"].items()})
PY
done

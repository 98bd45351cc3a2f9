# usage: bash tools/gpu_sweep.sh LIB VAR "v1 v2 ..."  -- serial bench per env value
mkdir -p gpurun_out
L=$1; V=$2
for x in $3; do
  env $V=$x REAX_LIBRARY=$PWD/$L REAX_SERIAL=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/sweep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); print('$V=$x', 'ms/step %.4f' % d['ms_per_step'], {k: round(v*1000,1) for k,v in d['kernel_ms_per_step'].items()})"
done

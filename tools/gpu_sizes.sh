# usage: bash tools/gpu_sizes.sh TAG -- bench at c1..c4 (device-only) + serial per-kernel times at c1
mkdir -p gpurun_out
TAG=${1:-sz}
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/size_${TAG}_c$c.json 2> gpurun_out/size_${TAG}_c$c.err
  REAX_SERIAL=1 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/size_${TAG}_serial_c$c.json 2>> gpurun_out/size_${TAG}_c$c.err
done
for f in gpurun_out/size_${TAG}_*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['config']['workload'], d['ms_per_step'], d['value']/1e6, d['kernel_ms_per_step'])"; done

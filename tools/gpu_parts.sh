python -m pytest tests/test_parity_gpu.py -q -x -m gpu -p no:cacheprovider -k "c0_full or c1_full or tiny or ragged or exact or outside or capacity or separate or graph or deterministic" 2>&1 | tail -1
for P in 1 2 3 4 6; do
  REAX_PARTS=$P timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "
import json; d=json.load(open('gpurun_out/p.json')); print('P=$P', 'ms/step %.4f' % d['ms_per_step'], '%.1fM' % (d['value']/1e6))" || tail -3 gpurun_out/p.err
done

bash tools/gpu_variants.sh paper_1706_07772_b200/libreax_minb2.so
for L in noflush nozero; do REAX_LIBRARY=$PWD/paper_1706_07772_b200/libreax_$L.so REAX_SERIAL=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/x.json')); print('$L', 'ms/step %.4f' % d['ms_per_step'], {k: round(v*1000,1) for k,v in d['kernel_ms_per_step'].items()})"; done
bash tools/gpu_sweep.sh paper_1706_07772_b200/libreax_minb2.so REAX_NBR_SPLIT "1 2 3 4 6 8"

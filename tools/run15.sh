for L in libreax libreax_localxj libreax_norow libreax_nomem libreax_nothing; do
 REAX_LIBRARY=$PWD/paper_1706_07772_b200/$L.so REAX_SERIAL=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/x.json 2>gpurun_out/x.err; python -c "
import json; d=json.load(open('gpurun_out/x.json')); print('$L', 'ms/step %.4f' % d['ms_per_step'], {k: round(v*1000,1) for k,v in d['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/x.err
done

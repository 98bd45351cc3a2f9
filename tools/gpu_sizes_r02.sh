# round-2 size sweep: bench line (device step, e2e, roofline) at c0..c4 with the final code
mkdir -p gpurun_out
for c in 0 1 2 3 4; do
  S=$([ $c -le 1 ] && echo 50 || echo 10)
  timeout 600 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline --no-next --no-c1 > gpurun_out/r02_size_c$c.json 2> gpurun_out/r02_size_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/r02_size_c$c.json')); print(d['config']['workload'][:40], round(d['ms_per_step'],4), round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(d['roofline']['frac'],3), round(d['roofline_kernels'][0]['frac'],3))"
done

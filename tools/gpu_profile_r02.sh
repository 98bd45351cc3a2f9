# round-2 evidence at c4 (bench workload): bench line, ncu launch list of the
# bench step, ncu --set full of k_nbr_build and k_nonbonded (c4), k_qeq_spmv (c3)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_c4.log 2>&1; tail -c 400 gpurun_out/r02_bench_c4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c1 --no-e2e --no-next > gpurun_out/r02_ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nbr_build -c 1 -o gpurun_out/r02_ncu_full_nbr_c4 -f \
  python tools/kbench.py 4 1 > gpurun_out/r02_ncu_nbr.log 2>&1; echo nbr rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nonbonded -c 1 -o gpurun_out/r02_ncu_full_nonbonded_c4 -f \
  python tools/kbench.py 4 1 > gpurun_out/r02_ncu_nb.log 2>&1; echo nb rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qeq_spmv -c 2 -o gpurun_out/r02_ncu_full_qeq_c3 -f \
  python tools/qeqbench.py 3 > gpurun_out/r02_ncu_qeq.log 2>&1; echo qeq rc=$?
timeout 300 python tools/qeqbench.py 3
timeout 300 python tools/qeqbench.py 4

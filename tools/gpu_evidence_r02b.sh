# round-2 final evidence (c4 bench workload): bench line (driver-like), c1 line,
# ncu launch lists, ncu --set full of k_nbr_build / k_nonbonded / the bond chain
# and finalize (c4) and k_qeq_spmv (c3)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench_c4.json 2> gpurun_out/r02b_bench_c4.err; tail -c 300 gpurun_out/r02b_bench_c4.json
timeout 600 python bench.py --config 1 --steps 50 --warmup 5 --no-cpu-baseline --no-next > gpurun_out/r02b_bench_c1.json 2> gpurun_out/r02b_bench_c1.err; echo c1 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c1 --no-e2e --no-next > gpurun_out/r02b_ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_c1.csv \
  python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline --no-c1 --no-e2e --no-next > gpurun_out/r02b_ncu_launch1.log 2>&1; echo launches1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nbr_build -c 1 -o gpurun_out/r02b_ncu_full_nbr_c4 -f \
  python tools/kbench.py 4 1 > gpurun_out/r02b_ncu_nbr.log 2>&1; echo nbr rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_nonbonded -c 1 -o gpurun_out/r02b_ncu_full_nonbonded_c4 -f \
  python tools/kbench.py 4 1 > gpurun_out/r02b_ncu_nb.log 2>&1; echo nb rc=$?
REAX_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cell_gather|k_bond_eval|k_bond_fill|k_bond_rank" -c 4 -o gpurun_out/r02b_ncu_full_chain_c4 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c1 --no-e2e --no-next > gpurun_out/r02b_ncu_chain.log 2>&1; echo chain rc=$?
REAX_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bond_delta|k_bond_correct|k_finalize" -c 3 -o gpurun_out/r02b_ncu_full_chain2_c4 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c1 --no-e2e --no-next > gpurun_out/r02b_ncu_chain2.log 2>&1; echo chain2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_qeq_spmv -c 2 -o gpurun_out/r02b_ncu_full_qeq_c3 -f \
  python tools/qeqbench.py 3 > gpurun_out/r02b_ncu_qeq.log 2>&1; echo qeq rc=$?

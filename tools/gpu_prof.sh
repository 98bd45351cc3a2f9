# usage: bash tools/gpu_prof.sh TAG  -- opbench + ncu --set full of the two window kernels on c1
set -x
TAG=${1:-prof}
mkdir -p gpurun_out
[ -n "$OPBENCH" ] && ./tools/opbench > gpurun_out/opbench.txt 2>&1; cat gpurun_out/opbench.txt
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_nbr_build|k_nonbonded}" -s ${KSKIP:-2} -c ${KCOUNT:-2} -o gpurun_out/$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log

# usage: bash tools/gpu_prof_lib.sh TAG LIB KREGEX  -- ncu --set full of one kernel launch (serial step) with a given library
set -x
TAG=$1; L=$2; K=${3:-k_nonbonded}
mkdir -p gpurun_out
REAX_LIBRARY=$PWD/$L REAX_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log

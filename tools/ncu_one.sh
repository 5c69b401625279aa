#!/bin/bash
# One `ncu --set full` capture of kernel $1 inside the C4 bench (after a
# plain run of the same command exited 0), raw + source pages as CSV.
#   tools/ncu_one.sh <kernel regex> <tag>
set -u
k=$1; tag=${2:-x}
python bench.py --steps 1 --warmup 1 --no-ras --no-cpu-baseline --no-spmv > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 2 -c 1 \
    -o gpurun_out/one_${tag} python bench.py --steps 1 --warmup 3 --no-ras \
    --no-cpu-baseline --no-spmv > gpurun_out/one_${tag}.log 2>&1
ncu -i gpurun_out/one_${tag}.ncu-rep --page raw --csv > gpurun_out/one_${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/one_${tag}.ncu-rep --page details --csv > gpurun_out/one_${tag}_details.csv 2>/dev/null
ncu -i gpurun_out/one_${tag}.ncu-rep --page source --csv > gpurun_out/one_${tag}_source.csv 2>/dev/null
rm -f gpurun_out/one_${tag}.ncu-rep

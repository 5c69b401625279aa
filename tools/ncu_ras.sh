#!/bin/bash
set -u
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmv > /dev/null 2>&1 || exit 1
for k in k_ilu_factor k_ilu_apply; do
ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 1 -c 1 \
    -o gpurun_out/one_$k python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-spmv > gpurun_out/one_$k.log 2>&1
ncu -i gpurun_out/one_$k.ncu-rep --page raw --csv > gpurun_out/one_${k}_raw.csv 2>/dev/null
ncu -i gpurun_out/one_$k.ncu-rep --page source --csv > gpurun_out/one_${k}_source.csv 2>/dev/null
rm -f gpurun_out/one_$k.ncu-rep
done

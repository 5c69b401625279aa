#!/bin/bash
# build variants on the GPU box and run the C4 bench (with the ras_exact leg)
#   tools/sweep_ras_flags.sh name1 "-DX=1" name2 "-DX=2" ...
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ISC_NVCC_EXTRA="$flags" python -m paper_1811_11992_b200.build > /dev/null || exit 1
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-spmv > gpurun_out/swr_$name.json 2> gpurun_out/swr_$name.err
done

#!/bin/bash
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ISC_NVCC_EXTRA="$flags" python -m paper_1811_11992_b200.build > /dev/null || exit 1
  python bench.py --precond ras --no-ras --no-cpu-baseline --no-spmv --steps 4 > gpurun_out/ras_$name.json 2> gpurun_out/ras_$name.err
done

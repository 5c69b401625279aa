#!/bin/bash
# occupancy sweep of the stencil passes (run on the GPU box)
for v in "$@"; do
  ISC_NVCC_EXTRA="-DMC_MINB=$v" python -m paper_1811_11992_b200.build > /dev/null || exit 1
  python bench.py --no-ras --no-cpu-baseline > gpurun_out/minb_$v.json 2> gpurun_out/minb_$v.err
done

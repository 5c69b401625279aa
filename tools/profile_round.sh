#!/bin/bash
# Round-end measurement on the GPU box: bench line, launch list, full ncu
# captures of the dominant kernels (each only after the plain run exits 0).
set -u
tag=${1:-r1}
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || exit 1
python bench.py --impl reference > gpurun_out/ref_$tag.json 2> gpurun_out/ref_$tag.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 1 --no-ras --no-cpu-baseline --no-spmv > gpurun_out/ncu_launch_$tag.log 2>&1
for k in k_cc6_red k_cc6_black k_sc_update_p k_sc_update_s k_sc_update_xr k_face_eval_light k_face_eval_energy k_face_gather k_decouple_compact_t k_cell_props k_cell_gas k_cell_rows k_mc_factor_cond_t k_cc_red_bc k_cc6_xred k_wells; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 2 -c 1 \
      -o gpurun_out/full_${tag}_$k python bench.py --steps 1 --warmup 3 --no-ras \
      --no-cpu-baseline --no-spmv > gpurun_out/ncu_full_${tag}_$k.log 2>&1
  rep=gpurun_out/full_${tag}_$k.ncu-rep
  ncu -i $rep --page raw --csv > gpurun_out/full_${tag}_${k}_raw.csv 2>/dev/null
  ncu -i $rep --page details --csv > gpurun_out/full_${tag}_${k}_details.csv 2>/dev/null
  ncu -i $rep --page source --csv > gpurun_out/full_${tag}_${k}_source.csv 2>/dev/null
  [ "$k" = k_cc6_black ] || rm -f $rep   # keep one report (gpurun_out <= 64 MiB)
done

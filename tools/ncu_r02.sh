#!/bin/bash
# Profiling pass for one round (run on the GPU box through gpurun; outputs land in gpurun_out/).
#  1. launch list of the bench's timed region (the same command the driver runs, kernels serialised and
#     cold-cached by ncu: per-launch shares, not absolute times)
#  2. launch list of one steady-state refresh iteration (iteration 200, timing from 20) with the size-class
#     bodies visible (TDPG_NO_COND=1)
#  3. one `--set full` capture of the GP kernels of a bench iteration (DRAM traffic, stalls, source)
TAG=${1:-r02}
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline \
    > gpurun_out/launches_${TAG}_bench.log 2>&1
TDPG_NO_COND=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_refresh.csv python tools/prof_refresh.py 200 1000000 20 > gpurun_out/launches_${TAG}_refresh.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"k_wa_axis_group|k_wa_generic|k_density_scatter|k_dens_grad|k_density_bins|k_cells|k_fin_" \
    -c 9 -o gpurun_out/full_${TAG} -f python tools/prof_refresh.py 5 > gpurun_out/full_${TAG}.log 2>&1
echo done

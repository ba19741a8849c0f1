#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (N=1), ncu launch list + one full capture.
# Usage (on the box): bash tools/gpu_round.sh [tag] [what...]   what ⊆ {tests,smoke,bench,launches,full}
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-tests smoke bench launches full}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi_$TAG.txt 2>&1
for w in $WHAT; do
  case $w in
    tests)  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?";;
    smoke)  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?";;
    bench)  timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_$TAG.json;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
               --log-file gpurun_out/launches_$TAG.csv python tools/prof_iter.py > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?";;
    full)   timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_wa|k_cells|k_dens}" \
               --profile-from-start off -c ${NCU_C:-8} -o gpurun_out/full_$TAG python tools/prof_iter.py > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?";;
  esac
done

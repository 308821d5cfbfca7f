#!/bin/bash
# Reproduce profiles/ on one B200 (run under gpurun from the repo root), then
# summarise here:   bash scripts/refresh_profiles.sh  &&  bash scripts/refresh_profiles.sh --summarise
set -e
if [ "$1" = "--summarise" ]; then
  tail -1 gpurun_out/bench.log > profiles/r01_bench.json
  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches_solve.md --last-solve > /dev/null
  cp gpurun_out/launches.csv profiles/r01_launches_solve.csv
  for c in 3 5; do
    python scripts/ncu_summary.py launches gpurun_out/launches_c$c.csv profiles/r01_launches_solve_c$c.md --last-solve > /dev/null
    cp gpurun_out/launches_c$c.csv profiles/r01_launches_solve_c$c.csv
  done
  python scripts/ncu_summary.py full gpurun_out/prof_full.ncu-rep profiles/r01_ncu_full_projectors.md profiles/ncu_traffic.json > /dev/null
  exit 0
fi
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.log 2>&1
# each ncu run only after the same command exited 0 without ncu (B200_PROFILING.md)
python bench.py --profile-once --no-detail --no-cpu > gpurun_out/plain1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --profile-once --no-detail --no-cpu > gpurun_out/ncu1.log 2>&1
for c in 3 5; do
  python scripts/profile_solve.py --cfg $c > gpurun_out/plain_c$c.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv \
        python scripts/profile_solve.py --cfg $c > gpurun_out/ncu_c$c.log 2>&1
done
python scripts/profile_run.py --mode kernels > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_backward" -s 1 -c 4 \
      -o gpurun_out/prof_full python scripts/profile_run.py --mode kernels > gpurun_out/ncu2.log 2>&1

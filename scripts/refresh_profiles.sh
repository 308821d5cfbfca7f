#!/bin/bash
# Reproduce profiles/ (round 2) on one B200 (run under gpurun from the repo
# root), then summarise here:
#   gpurun -- bash scripts/refresh_profiles.sh   &&   bash scripts/refresh_profiles.sh --summarise
# (profiles/parity_r02.md: run the GPU tests with MS2G_PARITY_LOG=gpurun_out/parity_r02.json first)
# Every ncu capture runs only after the same command exited 0 without ncu
# (B200_PROFILING.md); ncu timings are never bench values.  The projector
# capture is summarised into profiles/ncu_traffic.json on the box BEFORE the
# bench runs, so the bench line's roofline.binding / traffic come from the
# same kernel sources (source hash) as the bench itself.
set -e
R=r02
if [ "$1" = "--summarise" ]; then
  tail -1 gpurun_out/bench.log > profiles/${R}_bench.json
  tail -1 gpurun_out/bench_c5.log > profiles/${R}_bench_c5.json
  cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
  python scripts/ncu_summary.py full gpurun_out/prof_full.ncu-rep profiles/${R}_ncu_full_projectors.md > /dev/null
  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/${R}_launches_solve.md --last-solve > /dev/null
  cp gpurun_out/launches.csv profiles/${R}_launches_solve.csv
  for c in 3 5; do
    python scripts/ncu_summary.py launches gpurun_out/launches_c$c.csv profiles/${R}_launches_solve_c$c.md --last-solve > /dev/null
    cp gpurun_out/launches_c$c.csv profiles/${R}_launches_solve_c$c.csv
  done
  python scripts/ncu_summary.py full gpurun_out/prof_gather.ncu-rep profiles/${R}_ncu_full_adjoint_gather.md > /dev/null
  python scripts/ncu_summary.py full gpurun_out/prof_c5fwd.ncu-rep profiles/${R}_ncu_full_forward_batch8.md > /dev/null
  cp gpurun_out/adjoint_variants.log profiles/${R}_adjoint_variants.log
  python scripts/ncu_summary.py launches gpurun_out/launches_shard8.csv profiles/${R}_launches_shard8.md --last-solve > /dev/null
  cp gpurun_out/launches_shard8.csv profiles/${R}_launches_shard8.csv
  cp gpurun_out/tv_probe.log profiles/${R}_tv_probe.log
  if [ -f gpurun_out/parity_r02.json ]; then
    python scripts/parity_report.py gpurun_out/parity_r02.json profiles/parity_r02.md
  fi
  exit 0
fi
mkdir -p gpurun_out
python scripts/src_hash.py > gpurun_out/prof_hash.txt
python scripts/profile_run.py --mode kernels > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_backward" -s 1 -c 4 \
      -o gpurun_out/prof_full -f python scripts/profile_run.py --mode kernels > gpurun_out/ncu2.log 2>&1
python scripts/ncu_summary.py full gpurun_out/prof_full.ncu-rep gpurun_out/ncu_full_projectors.md \
    profiles/ncu_traffic.json > /dev/null
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
python bench.py --cfg 5 --steps 10 --warmup 3 > gpurun_out/bench_c5.log 2>&1
python bench.py --profile-once --no-detail --no-cpu > gpurun_out/plain1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --profile-once --no-detail --no-cpu > gpurun_out/ncu1.log 2>&1
for c in 3 5; do
  python scripts/profile_solve.py --cfg $c > gpurun_out/plain_c$c.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$c.csv \
        python scripts/profile_solve.py --cfg $c > gpurun_out/ncu_c$c.log 2>&1
done
python scripts/adjoint_variants.py > gpurun_out/adjoint_variants.log 2>&1
python scripts/profile_small.py shard > gpurun_out/plain5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_shard8.csv \
      python scripts/profile_small.py shard > gpurun_out/ncu5.log 2>&1
python scripts/tv_probe.py > gpurun_out/tv_probe.log 2>&1
MS2G_BP_VARIANT=gather python scripts/profile_run.py --mode kernels > gpurun_out/plain3.log 2>&1 && \
  MS2G_BP_VARIANT=gather ncu --set full --clock-control none --import-source on -k regex:"k_backward_gather" -s 1 \
      -c 1 -o gpurun_out/prof_gather -f python scripts/profile_run.py --mode kernels > gpurun_out/ncu3.log 2>&1
python scripts/profile_solve.py --cfg 5 > gpurun_out/plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_forward_batch" -s 2 -c 1 \
      -o gpurun_out/prof_c5fwd -f python scripts/profile_solve.py --cfg 5 > gpurun_out/ncu4.log 2>&1

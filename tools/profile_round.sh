#!/bin/bash
# Round profile capture on one B200 (run under gpurun from the repo root):
#   1. the bench line (no profiler attached),
#   2. the launch list of a short bench run (per-launch device times),
#   3. one `ncu --set full` capture of each steady-state kernel of the
#      default fixed-step structure (S12 and S3).
# Usage: bash tools/profile_round.sh <tag>
set -e
tag=${1:-r}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_$tag.log 2>&1
ncu --set full --import-source on --clock-control none -k 'regex:s12' -c 1 \
    -o gpurun_out/s12_$tag python tools/prof_stage.py 8192 4 > gpurun_out/ncu_s12_$tag.log 2>&1
ncu --set full --import-source on --clock-control none -k sgn_stage_kernel --launch-skip 1 -c 1 \
    -o gpurun_out/s3_$tag python tools/prof_stage.py 8192 4 > gpurun_out/ncu_s3_$tag.log 2>&1
echo done

#!/bin/bash
# Round-2 evidence pass on one B200 (run under gpurun from the repo root):
# GPU tests, smoke, bench lines (config 4, reflecting, 1-rank NCCL ring,
# adaptive), the reference arm, a launch list and ncu --set full captures of
# S12 / S3 (periodic) and S12 (walls).
tag=${1:-r2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$tag.log 2>&1; echo tests=$?; tail -1 gpurun_out/gputests_$tag.log
python __graft_entry__.py > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
timeout 400 python bench.py --bc reflecting --no-cpu-baseline > gpurun_out/bench_refl_$tag.json 2>/dev/null; echo refl=$?
timeout 400 python bench.py --slab-ring --no-cpu-baseline > gpurun_out/bench_ring_$tag.json 2>/dev/null; echo ring=$?
timeout 300 python bench.py --adaptive 1e-8 --steps 50 > gpurun_out/bench_adapt_$tag.json 2>/dev/null; echo adapt=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>/dev/null; echo ref=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --sustained 0 > /dev/null 2>&1; echo launches=$?
timeout 300 ncu --set full --import-source on --clock-control none -k "regex:s12" -c 1 -o gpurun_out/s12_$tag python tools/prof_stage.py 8192 4 > /dev/null 2>&1; echo ncu_s12=$?
timeout 300 ncu --set full --import-source on --clock-control none -k "regex:sgn_stage_kernel" --launch-skip 1 -c 1 -o gpurun_out/s3_$tag python tools/prof_stage.py 8192 4 > /dev/null 2>&1; echo ncu_s3=$?
timeout 300 ncu --set full --import-source on --clock-control none -k "regex:s12" -c 1 -o gpurun_out/s12w_$tag python tools/prof_stage.py 8192 4 0 - walls > /dev/null 2>&1; echo ncu_s12w=$?
# text exports of the captures (the gpurun copy-back is capped at 64 MiB): keep
# the S12 report, export and drop the others
for r in s12 s3 s12w; do
  f=gpurun_out/${r}_$tag.ncu-rep
  [ -f $f ] || continue
  ncu -i $f --page raw --csv > gpurun_out/${r}_${tag}_raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > gpurun_out/${r}_${tag}_src.csv 2>/dev/null
  [ $r != s12 ] && rm -f $f
done
du -sh gpurun_out

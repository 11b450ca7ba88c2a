set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2b.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests_r2b.log
python __graft_entry__.py > gpurun_out/smoke_r2b.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench=$?
timeout 400 python bench.py --bc reflecting --no-cpu-baseline > gpurun_out/bench_refl_r2b.json 2> gpurun_out/bench_refl_r2b.err; echo refl=$?
timeout 400 python bench.py --slab-ring --no-cpu-baseline > gpurun_out/bench_ring_r2b.json 2> gpurun_out/bench_ring_r2b.err; echo ring=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --sustained 0 > gpurun_out/launches_r2b.log 2>&1; echo launches=$?
timeout 300 ncu --set full --import-source on --clock-control none -k "regex:s12" -c 1 -o gpurun_out/s12_r2b python tools/prof_stage.py 8192 4 > /dev/null 2>&1; echo ncu1=$?
timeout 300 ncu --set full --import-source on --clock-control none -k "regex:sgn_stage_kernel" --launch-skip 1 -c 1 -o gpurun_out/s3_r2b python tools/prof_stage.py 8192 4 > /dev/null 2>&1; echo ncu2=$?

#!/bin/bash
# Round-2 session-4 evidence run (one B200): GPU suite, smoke, default bench (with the
# CPU baseline leg), reference arm, configs[3] / FP32 configs[4] shard benches,
# launch list of the default command. Outputs under gpurun_out/ (small files only).
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/r02s4f_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02s4f_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02s4f_smoke.log 2>&1; echo "smoke rc=$?" >> $O/r02s4f_smoke.log
timeout 900 python bench.py > $O/r02s4f_bench_default.json 2> $O/r02s4f_bench_default.err
timeout 900 python bench.py --impl reference > $O/r02s4f_bench_ref.json 2> /dev/null
timeout 900 python bench.py --config E4f32 --no-cpu > $O/r02s4f_bench_E4f32.json 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02s4f_launches_B.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la $O

#!/bin/bash
# Round-2 session-3 evidence run (one B200). part 1: benches + launch list; part 2 (arg "ncu"): ncu.
O=gpurun_out
if [ "$1" = "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemv_fwd" -c 1 -o $O/r02s3_gemv_fwd_B python bench.py --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:"k_r2c_fast|k_c2r_fast" -c 2 -o $O/r02s3_fft_C python bench.py --config C --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1
  ls -la $O; exit 0
fi
timeout 600 python bench.py > $O/r02s3_bench_B.json 2> $O/r02s3_bench_B.err
timeout 900 python bench.py --config D --no-cpu > $O/r02s3_bench_D.json 2> /dev/null
timeout 900 python bench.py --config C --no-cpu > $O/r02s3_bench_C.json 2> /dev/null
timeout 900 python bench.py --config E8 --no-cpu > $O/r02s3_bench_E8.json 2> /dev/null
timeout 900 python bench.py --config E4f32 --no-cpu > $O/r02s3_bench_E4f32.json 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02s3_launches_B.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
ls -la $O

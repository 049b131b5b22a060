#!/bin/bash
# Round-2 evidence run (one B200): benches, launch lists, ncu of the new kernels.
set -x
O=gpurun_out
timeout 600 python bench.py > $O/r02s2_bench_B.json 2> $O/r02s2_bench_B.err
timeout 900 python bench.py --config D --no-cpu > $O/r02s2_bench_D.json 2> $O/r02s2_bench_D.err
timeout 600 python bench.py --impl reference > $O/r02s2_bench_ref.json 2> $O/r02s2_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02s2_launches_B.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02s2_launches_D.csv python bench.py --config D --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c_tma|k_c2r_tma" -c 2 -o $O/r02s2_fft_D python bench.py --config D --steps 1 --warmup 0 --no-cpu > $O/ncu_fft_D.log 2>&1
MASTER_ADDR=127.0.0.1 BTG_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --config Bp > $O/r02s2_bench_gloo2.json 2> $O/r02s2_bench_gloo2.err
ls -la $O

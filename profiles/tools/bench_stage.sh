#!/bin/bash
# bench.py one config, printing step ms, per-stage ms and e2e ms (dev tool).
#   profiles/tools/bench_stage.sh D [env assignments...]
cfg=$1; shift
env "$@" timeout 900 python bench.py --config "$cfg" --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $*', round(d['ms_per_step'],3), {k:{s:round(v,3) for s,v in x.items()} for k,x in d['roofline']['stage_ms'].items()}, 'e2e', d.get('e2e',{}).get('ms_per_step'))"

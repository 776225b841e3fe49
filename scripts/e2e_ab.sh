#!/bin/bash
# A/B of an env setting on the end-to-end (pinned host x / y) number of bench.py:
#   bash scripts/e2e_ab.sh c4 "HMAT_PDL=3"
set -u
cfg=$1
envset=$2
for rep in 1 2; do
  for mode in base new; do
    if [ $mode = new ]; then e="env $envset"; else e=""; fi
    $e python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']
print('$mode', round(d['value'],2), 'e2e', round(e['value'],2), [round(v,3) for v in e['runs_ms_per_step']], 'blocking', round(e['blocking']['value'],2))"
  done
done

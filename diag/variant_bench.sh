#!/bin/bash
# device-timed bench value (60 steps) of each variant: diag/variant_bench.sh base v1 base v1 ...
for v in "$@"; do
  if [ "$v" = base ]; then unset GSMAP_B200_VARIANT; else export GSMAP_B200_VARIANT=$v; fi
  timeout 300 python bench.py --steps 60 --warmup 6 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'])"
done

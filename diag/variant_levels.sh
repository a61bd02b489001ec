#!/bin/bash
# per-level blend kernel times of each built variant (and the product build), from the bench's
# profile pass: diag/variant_levels.sh base fwd6 bwd12 ...
for v in "$@"; do
  if [ "$v" = base ]; then unset GSMAP_B200_VARIANT; else export GSMAP_B200_VARIANT=$v; fi
  timeout 200 python bench.py --profile-only --steps 9 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['per_level_kernel_ms']
print('$v', d['value'], ' '.join(f\"{l}: fwd {k[l]['blend_fwd']:.3f} bwd {k[l]['blend_bwd']:.3f} tot {sum(k[l].values()):.3f}\" for l in ('L2','L1','L0')))"
done

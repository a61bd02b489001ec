#!/bin/bash
# per-level kernel-family times of each built variant (and the product build), from the bench's
# profile pass: diag/variant_levels.sh base fwd6 bwd12 ...
for v in "$@"; do
  if [ "$v" = base ]; then unset GSMAP_B200_VARIANT; else export GSMAP_B200_VARIANT=$v; fi
  timeout 200 python bench.py --profile-only --steps 9 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['per_level_kernel_ms']
short={'preprocess_fwd':'k1','depth_sort_pack_scan':'dsort','tile_keys_sort_ranges':'tsort','blend_fwd':'fwd',
       'loss_l1_ssim_depth':'loss','blend_bwd':'bwd','preprocess_bwd':'k8','adam':'adam'}
print('$v', d['value'])
for l in ('L2','L1','L0'):
    print('   ', l, ' '.join(f'{short.get(n,n)} {t:.3f}' for n,t in k[l].items()), f'tot {sum(k[l].values()):.3f}')"
done

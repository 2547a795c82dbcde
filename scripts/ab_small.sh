#!/bin/bash
# A/B of the compact NTT pass policy (HC_NTT_SMALL = 0 off, 1 lone sub-wave launches, 2 every sub-wave launch, 3 every launch)
O=gpurun_out/ab_small
mkdir -p $O
for v in ${POLICIES:-0 1 3}; do
  HC_NTT_SMALL=$v python bench.py --workload softmax --steps 5 --no-cpu > $O/softmax_$v.json 2>$O/softmax_$v.err
  HC_NTT_SMALL=$v python bench.py --no-cpu --steps 10 > $O/pair_$v.json 2>$O/pair_$v.err
  HC_NTT_SMALL=$v python bench.py --workload train --steps 3 --no-cpu > $O/train_$v.json 2>$O/train_$v.err
done
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_small/*.json')):
    try:
        d=json.load(open(f)); print(f, round(d['value'],3), {k:v for k,v in d['kernel_breakdown_ms'].items() if 'ntt' in k})
    except Exception as e: print(f, 'ERR', e)
P

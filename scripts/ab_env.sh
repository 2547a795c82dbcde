#!/bin/bash
# A/B of one environment knob on the pair, softmax and the level-12 rotation probe: ab_env.sh VAR v0 v1 ...
VAR=$1; shift
O=gpurun_out/ab_$VAR
mkdir -p $O
for v in "$@"; do
  env $VAR=$v python bench.py --no-cpu --steps 10 > $O/pair_$v.json 2>$O/pair_$v.err
  env $VAR=$v python bench.py --workload softmax --steps 5 --no-cpu > $O/softmax_$v.json 2>$O/softmax_$v.err
  env $VAR=$v python scripts/ks_batch_probe.py 3 8 > $O/ks3_$v.log 2>&1
done
python - "$O" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/*.json')):
    try:
        d=json.load(open(f)); kb=d['kernel_breakdown_ms']; print(f, round(d['value'],3), {k:kb[k] for k in list(kb)[:6]})
    except Exception as e: print(f, 'ERR', e)
P
grep -H "key switches" $O/ks3_*.log

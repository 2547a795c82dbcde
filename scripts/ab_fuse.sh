#!/bin/bash
# A/B of the one-launch (cooperative) forms of a lone INTT / rescale: "INTT_MAX RS_MAX" pairs
O=gpurun_out/ab_fuse
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "per_op or fused_ops or other_rings or config3_softmax or nag_steps or softmax_small12 or adversarial" > $O/parity.log 2>&1
tail -n 3 $O/parity.log
for cfg in "0 0" "9 0" "9 18" "13 24" "6 10"; do
  set -- $cfg
  tag=i$1_r$2
  HC_INTT_FUSE=$1 HC_RS_FUSE=$2 timeout 600 python bench.py --workload softmax --steps 5 --no-cpu > $O/softmax_$tag.json 2>$O/softmax_$tag.err
  HC_INTT_FUSE=$1 HC_RS_FUSE=$2 timeout 600 python bench.py --workload train --steps 3 --no-cpu > $O/train_$tag.json 2>$O/train_$tag.err
done
python - "$O" <<'P'
import json,glob,sys
for f in sorted(glob.glob(sys.argv[1]+'/*.json')):
    try:
        d=json.load(open(f)); kb=d['kernel_breakdown_ms']; print(f, round(d['value'],3), {k:kb[k] for k in kb if 'ntt_inv' in k or 'rs_' in k})
    except Exception as e: print(f, 'ERR', e)
P

#!/bin/bash
# pair ms over (key switches per batched pipeline) x (concurrent streams)
O=gpurun_out/sweep
mkdir -p $O
for b in 2 3 4 6 8; do for s in 2 3 4 6; do
  HC_BATCH=$b HC_STREAMS=$s python bench.py --no-cpu --steps 10 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('batch',$b,'streams',$s,'pair',round(d['value'],3),'abt',round(d['diag_abt_ms'],3),'atb',round(d['diag_atb_ms'],3))" | tee -a $O/pair_sweep.txt
done; done

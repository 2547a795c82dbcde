#!/bin/bash
# ncu --set full of one lone level-12 rotation (batch 1) under the compact-pass policy given as $1 (default 1)
V=${1:-1}
O=gpurun_out/lone
mkdir -p $O
HC_NTT_SMALL=$V python scripts/ks_batch_probe.py 1 2 > $O/probe_$V.log 2>&1
HC_NTT_SMALL=$V HC_PROBE_PROFILE=1 ncu --set full --clock-control none --profile-from-start off -f -o $O/lone_$V \
    python scripts/ks_batch_probe.py 1 2 > $O/ncu_$V.log 2>&1
python scripts/ncu_summary.py $O/lone_$V.ncu-rep > $O/lone_${V}_summary.txt
rm -f $O/lone_$V.ncu-rep
cat $O/probe_$V.log
cut -c1-330 $O/lone_${V}_summary.txt | head -9

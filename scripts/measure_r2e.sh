#!/bin/bash
# Final measurement of round 2 (compact NTT pass for chain launches) on one B200:
# bench lines, launch list of the bench command, ncu --set full of the batched
# rotation pipeline and of one radix-4 ladder stage.  Every command runs alone
# first without ncu.
O=gpurun_out/r2e
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo exit=$? >> $O/gputest.log
python bench.py > $O/bench_pair.json 2> $O/bench_pair.err
python bench.py --workload softmax --steps 5 --no-cpu > $O/softmax.json 2>/dev/null
python bench.py --workload train --steps 3 --no-cpu > $O/train.json 2>/dev/null
python bench.py --workload table4 --no-cpu > $O/table4.json 2>/dev/null
python bench.py --workload bootstrap --no-cpu > $O/bootstrap.json 2>/dev/null
python bench.py --workload softmax --boot ckks --steps 2 --warmup 1 --no-cpu > $O/softmax_ckks.json 2>/dev/null
python bench.py --workload train --boot ckks --steps 1 --warmup 1 --no-cpu > $O/train_ckks.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > $O/reference.json 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_exit=$? >> $O/smoke.log
python scripts/ks_batch_probe.py 3 2 > $O/ks_probe.log 2>&1
HC_PROBE_PROFILE=1 ncu --set full --clock-control none --profile-from-start off -o $O/ks_batch3 \
    python scripts/ks_batch_probe.py 3 2 > $O/ncu_ks.log 2>&1
ncu -i $O/ks_batch3.ncu-rep --page raw --csv > $O/ks_batch3_raw.csv
python scripts/ncu_summary.py $O/ks_batch3.ncu-rep > $O/ks_batch3_summary.txt
python scripts/ncu_ks_evidence.py $O/ks_batch3_raw.csv 9 $O/ncu_keyswitch.json 1 94370000 "ncu --set full of 9 level-12 rotations (cfg1) in batched pipelines of 3 (scripts/ks_batch_probe.py 3 2: warm-up pipeline + 2 measured), serialised, cold cache" > /dev/null
python scripts/ladder_probe.py 3 2 2 1 11 > $O/ladder_probe.log 2>&1
HC_PROBE_PROFILE=1 ncu --set full --clock-control none --profile-from-start off -o $O/ladder_stage3 \
    python scripts/ladder_probe.py 3 2 2 1 11 > $O/ncu_ladder.log 2>&1
ncu -i $O/ladder_stage3.ncu-rep --page raw --csv > $O/ladder_stage3_raw.csv
python scripts/ncu_summary.py $O/ladder_stage3.ncu-rep > $O/ladder_stage3_summary.txt
python scripts/ncu_ks_evidence.py $O/ladder_stage3_raw.csv 9 $O/ncu_ladder.json 2 110100480 \
    "ncu --set full of 9 radix-4 rotate-and-sum stages (18 doubling steps: warm-up + 2 measured) at level 11 (cfg1) in batched pipelines of 3 (scripts/ladder_probe.py 3 2 2 1 11), serialised, cold cache" > /dev/null
rm -f $O/*.ncu-rep
gzip -f $O/ks_batch3_raw.csv $O/ladder_stage3_raw.csv
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 7000 -c 3000 --csv --log-file $O/launches.csv \
    python bench.py --no-cpu --steps 1 --warmup 3 > $O/ncu_launch.log 2>&1
python scripts/launch_summary.py $O/launches.csv > $O/launch_summary.txt
gzip -f $O/launches.csv
echo done

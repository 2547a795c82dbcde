#!/bin/bash
# Final lines of round 2 (batched schedule ops, 6 key switches per pipeline): tests, bench lines, smoke, reference arm, launch list of the bench command.
O=gpurun_out/r2m
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; echo exit=$? >> $O/gputest.log
python bench.py > $O/bench_pair.json 2> $O/bench_pair.err
python bench.py --workload softmax --steps 5 --no-cpu > $O/softmax.json 2>/dev/null
python bench.py --workload train --steps 3 --no-cpu > $O/train.json 2>/dev/null
python bench.py --workload table4 --no-cpu > $O/table4.json 2>/dev/null
python bench.py --workload bootstrap --no-cpu > $O/bootstrap.json 2>/dev/null
python bench.py --workload train --boot ckks --steps 1 --warmup 1 --no-cpu > $O/train_ckks.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > $O/reference.json 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_exit=$? >> $O/smoke.log
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 5000 -c 3000 --csv --log-file $O/launches.csv \
    python bench.py --no-cpu --steps 1 --warmup 3 > $O/ncu_launch.log 2>&1
python scripts/launch_summary.py $O/launches.csv > $O/launch_summary.txt
gzip -f $O/launches.csv
tail -n 2 $O/gputest.log; tail -n 1 $O/smoke.log

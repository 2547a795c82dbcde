#!/bin/bash
# End-of-session measurement on one B200: bench lines (pair, softmax, training
# step, reference arm), the launch list of the bench command, and one
# ncu --set full capture of the key-switch kernels of a batched pipeline.
# Every command runs alone first without ncu.
O=gpurun_out/final
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest_exit=$? >> $O/pytest_gpu.log
python bench.py > $O/bench_pair.json 2> $O/bench_pair.err
python bench.py --workload softmax --steps 5 > $O/softmax.json 2>/dev/null
python bench.py --workload train --steps 3 > $O/train.json 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > $O/reference.json 2>/dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_exit=$? >> $O/smoke.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --no-cpu --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
gzip -f $O/launches.csv
python scripts/ks_batch_probe.py 3 4 > $O/ks_probe.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ks_ --launch-skip 8 -c 4 \
    -o $O/ks_full python scripts/ks_batch_probe.py 3 4 > $O/ncu_full.log 2>&1
echo done

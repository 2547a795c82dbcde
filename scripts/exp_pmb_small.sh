# NTT_PMB_SMALL experiment: softmax (chain), pair (headline) and training step with the in-tree build
set -e
python bench.py --no-cpu --workload softmax --steps 10 > gpurun_out/sm_chain.json 2>/dev/null
python bench.py --no-cpu > gpurun_out/pair_chain.json 2>/dev/null
python bench.py --no-cpu --workload train --steps 3 > gpurun_out/train_chain.json 2>/dev/null
python -c "import json;a=json.load(open('gpurun_out/sm_chain.json'));b=json.load(open('gpurun_out/pair_chain.json'));c=json.load(open('gpurun_out/train_chain.json'));print('chain', a['value'], b['value'], b['e2e']['value'], c['value'])"
python -m pytest tests -m gpu -x -q 2>&1 | tail -1

# MD_MINB_CHAIN experiment: resident-CTA budget of a lone key switch's ModDown chunk pass
run() { tag=$1; python bench.py --no-cpu --workload softmax --steps 10 > gpurun_out/sm_$tag.json 2>/dev/null; python bench.py --no-cpu > gpurun_out/pair_$tag.json 2>/dev/null; python -c "import json;a=json.load(open('gpurun_out/sm_$tag.json'));b=json.load(open('gpurun_out/pair_$tag.json'));print('$tag', a['value'], b['value'], b['e2e']['value'])"; }
run base
for v in 4 3; do touch paper_2403_14111_b200/csrc/keyswitch.cu; make -s -j8 -C paper_2403_14111_b200/csrc EXTRA=-DMD_MINB_CHAIN=$v > /dev/null 2>&1 || exit 9; run md$v; python -m pytest tests -m gpu -x -q -k "softmax or keyswitch or rotate" 2>&1 | tail -1; done

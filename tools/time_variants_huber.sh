#!/bin/bash
# A/B timing of libdbag.so variants (tools/build_variants.py), run on the GPU box:
#   bash tools/time_variants_huber.sh variant...
for v in "$@"; do
DBAG_LIB=paper_1708_07954_b200/_variants/$v.so python bench.py --config 5 --steps 10 --warmup 3 --no-cpu --loss huber > gpurun_out/hub_$v.json 2>gpurun_out/hub_$v.err
python -c "import json;d=json.loads(open('gpurun_out/hub_$v.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'], d['kernels']['local']['ms'], d['other_numerics']['ms_per_step'])"
done

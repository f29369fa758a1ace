#!/bin/bash
# A/B timing of libdbag.so variants (tools/build_variants.py), run on the GPU box:
#   bash tools/time_variants_huber_fast.sh variant...
for v in "$@"; do
DBAG_LIB=paper_1708_07954_b200/_variants/$v.so python bench.py --config 5 --steps 10 --warmup 3 --no-cpu --loss huber --numerics fast > gpurun_out/hubf_$v.json 2>gpurun_out/hubf_$v.err
python -c "import json;d=json.loads(open('gpurun_out/hubf_$v.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'], d['kernels']['local']['ms'])"
done

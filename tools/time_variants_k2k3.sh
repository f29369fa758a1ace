#!/bin/bash
# A/B timing of libdbag.so variants (tools/build_variants.py), run on the GPU box:
#   bash tools/time_variants_k2k3.sh variant...
for v in "$@"; do
DBAG_LIB=paper_1708_07954_b200/_variants/$v.so timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu > gpurun_out/k2_$v.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/k2_$v.log').read().strip().splitlines()[-1]);print('$v', 'point %.3f camera %.3f local %.3f'%(d['kernels']['point']['ms'], d['kernels']['camera']['ms'], d['kernels']['local']['ms']))"
done

#!/bin/bash
# A/B timing of libdbag.so variants (tools/build_variants.py), run on the GPU box:
#   bash tools/time_variants_blocks.sh variant...
for v in "$@"; do
for ppb in 32 8; do
DBAG_LIB=paper_1708_07954_b200/_variants/$v.so python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --points-per-block $ppb > gpurun_out/blk_${v}_$ppb.json 2>gpurun_out/blk_${v}_$ppb.err
python -c "import json;d=json.loads(open('gpurun_out/blk_${v}_$ppb.json').read().strip().splitlines()[-1]);print('$v ppb $ppb', '%.4g'%d['value'], d['ms_per_step'], d['counters']['n_trial'])"
done
done

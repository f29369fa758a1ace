#!/bin/bash
# usage: tools/time_variants.sh <config> <numerics> <steps> variant...
# A/B timing of paper_1708_07954_b200/_variants/<variant>.so (tools/build_variants.py):
# bench value and the per-kernel split (K1 local, K3 camera, K2 point) per round.
cfg=$1; num=$2; steps=$3; shift 3
for v in "$@"; do
  DBAG_LIB=paper_1708_07954_b200/_variants/$v.so timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --no-legs --numerics $num $BENCH_EXTRA > gpurun_out/var_${v}_${num}_c${cfg}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/var_${v}_${num}_c${cfg}.log').read().strip().splitlines()[-1]);k=d['kernels'];print('$v $num c$cfg', 'value %.4g'%d['value'], 'ms/round %.3f'%d['ms_per_step'], 'k1 %.3f k3 %.3f k2 %.3f'%(k['local']['ms'],k['camera']['ms'],k['point']['ms']), 'ns/trial %.4f'%(k['local']['ms']*1e6*d['steps']/max(1,d['counters']['n_trial'])))" 2>&1 | tail -1
done

#!/bin/bash
# usage: tools/time_variants.sh <config> <numerics> <steps> variant...
cfg=$1; num=$2; steps=$3; shift 3
for v in "$@"; do
  DBAG_LIB=paper_1708_07954_b200/_variants/$v.so timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --numerics $num > gpurun_out/var_${v}_${num}_c${cfg}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/var_${v}_${num}_c${cfg}.log').read().strip().splitlines()[-1]);print('$v $num c$cfg', 'value %.4g'%d['value'], 'k1 ms %.3f'%d['kernels']['local']['ms'], 'ns/trial %.4f'%(d['kernels']['local']['ms']*1e6*d['steps']/max(1,d['counters']['n_trial'])), 'trials %d'%d['counters']['n_trial'])" 2>&1 | tail -1
done

bash tools/time_variants.sh 5 exact 10 cur k1_stage k1_rollt k1_stage_rollt cur k1_stage k1_rollt k1_stage_rollt
for v in cur k1_stage k1_rollt k1_stage_rollt; do python - <<PY
import json
d=json.loads(open('gpurun_out/var_${v}_exact_c5.log').read().strip().splitlines()[-1]); print('$v', d['last_round']['max_primal_x'], d['last_round']['max_primal_y'], d['last_round']['max_dual_x'])
PY
done
bash tools/time_variants.sh 3 exact 10 cur k1_stage k1_rollt k1_stage_rollt
echo "== parity with k1_stage_rollt"
DBAG_LIB=paper_1708_07954_b200/_variants/k1_stage_rollt.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3

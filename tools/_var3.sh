bash tools/time_variants.sh 5 exact 10 cur k1_async cur k1_async
for v in cur k1_async; do python - <<PY
import json
d=json.loads(open('gpurun_out/var_${v}_exact_c5.log').read().strip().splitlines()[-1]); print('$v', d['last_round'])
PY
done
bash tools/time_variants.sh 2 exact 20 cur k1_async
bash tools/time_variants.sh 3 exact 10 cur k1_async
for v in hub_fixed3 cur; do
  echo "== $v"; DBAG_LIB=paper_1708_07954_b200/_variants/$v.so timeout 600 python tools/time_huber.py 5 10 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_local_per_round'], d['checksum'])"
done
echo "== parity with k1_async"
DBAG_LIB=paper_1708_07954_b200/_variants/k1_async.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5

for v in cur hub_u2 hub_u4 cur hub_u2; do
  echo "== $v"; DBAG_LIB=paper_1708_07954_b200/_variants/$v.so timeout 600 python tools/time_huber.py 5 10 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_local_per_round'], d['checksum'])"
done

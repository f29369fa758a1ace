import sys, time, os
sys.path.insert(0, os.getcwd())
import paper_1708_07954_b200 as P
s = P.generate_config_scene(2, 0)
for rep in range(3):
    t0 = time.perf_counter()
    g = P.AdmmSolver(s.problem, s.init, P.AdmmOptions(max_iters=100))
    t1 = time.perf_counter()
    tr = g.run()
    t2 = time.perf_counter()
    c = g.consensus()
    t3 = time.perf_counter()
    g.close()
    print(f"graph_off={os.environ.get('DBAG_NO_GRAPH')} rep {rep}: create {t1-t0:.3f}s run {t2-t1:.3f}s "
          f"consensus {t3-t2:.3f}s; sum wall_ms {sum(r['wall_ms'] for r in tr):.1f}", flush=True)

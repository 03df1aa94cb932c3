"""One COMPLETE sigma of the reference algorithm (blocked contract_sigma restatement, every
intermediate alpha row) on all host threads — validates bench.py's bounded-sample extrapolation.

    python tools/cpu_full_sigma.py [c4] [threads]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
cr = bench.CpuReference(cfg, int(sys.argv[2]) if len(sys.argv) > 2 else None)
rpt_probe, t_probe = cr.calibrate(cr.threads, 10.0)
rows_probe = cr.threads
per = -(-cr.na // cr.threads)  # ceil: every intermediate row exactly once across the threads
t0 = time.perf_counter()
t = cr.sample(cr.threads, per)[0]
wall = time.perf_counter() - t0
out = {"config": cfg, "threads": cr.threads, "rows_per_thread": per, "n_alpha": cr.na,
       "full_sigma_seconds": t, "wall_seconds": wall,
       "probe": {"rows": rows_probe, "seconds": t_probe, "extrapolated_full_sigma_seconds": t_probe * cr.na / rows_probe},
       "host": cr.info}
print(json.dumps(out), flush=True)
cr.close()

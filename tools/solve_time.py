"""Device time of one solve (L2 scrubbed) for configs under env variants (development aid)."""
import json, os, subprocess, sys
CODE = r'''
import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib
P = rq.baseline_config(sys.argv[1], device=True)
op = rq.build_operator(P, -0.5)
ms = C.c_double()
_lib.check(_lib.lib.rq_operator_time(op._h, 1 | 0x100, 20, 0, C.byref(ms)))
print(ms.value)
'''
cfg = sys.argv[1]
for var in sys.argv[2:] or [""]:
    env = dict(os.environ)
    for kv in filter(None, var.split(",")):
        k, v = kv.split("="); env[k] = v
    r = subprocess.run([sys.executable, "-c", CODE, cfg], env=env, capture_output=True, text=True)
    out = r.stdout.strip().splitlines()
    print(json.dumps({"cfg": cfg, "env": var, "solve_ms": float(out[-1]) if r.returncode == 0 and out else None,
                      "err": r.stderr[-300:] if r.returncode else ""}), flush=True)

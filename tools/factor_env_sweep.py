"""Factor time under environment variants (development aid): each variant in a
fresh process. Usage: factor_env_sweep.py cfg "VAR=a,VAR2=b" "VAR=c" ..."""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, ctypes as C
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib
P = rq.baseline_config(sys.argv[1], device=True)
o = rq.nested_dissection_order(P)
op = rq.build_operator(P, -0.5, o)
ms = C.c_double()
_lib.check(_lib.lib.rq_operator_time(op._h, 5 | 0x100, 3, 0, C.byref(ms)))
_lib.check(_lib.lib.rq_operator_time(op._h, 5 | 0x100, 10, 0, C.byref(ms)))
print(ms.value)
'''
cfg = sys.argv[1]
for var in sys.argv[2:] or [""]:
    env = dict(os.environ)
    for kv in filter(None, var.split(",")):
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CODE, cfg], env=env, capture_output=True, text=True)
    out = r.stdout.strip().splitlines()
    print(json.dumps({"cfg": cfg, "env": var, "ms": float(out[-1]) if r.returncode == 0 and out else None,
                      "err": r.stderr[-300:] if r.returncode else ""}), flush=True)

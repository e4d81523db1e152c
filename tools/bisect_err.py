import sys, ctypes as C, numpy as np, time
sys.path.insert(0,'.')
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib
def prof(tag, fh):
    ms=np.zeros(7); cnt=np.zeros(7,np.int64); w=np.zeros(7)
    try:
        _lib.check(_lib.lib.rq_factor_profile(fh, ms, cnt, w)); print(tag,'ok', ms.round(3), flush=True)
    except Exception as e: print(tag,'ERR',e, flush=True)
cfg=sys.argv[1]
P=rq.baseline_config(cfg, device=True); o=rq.nested_dissection_order(P); op=rq.build_operator(P,-0.5,o)
fh=_lib.lib.rq_operator_factor(op._h)
prof('A fresh', fh)
prof('A2 again', fh)
ms=C.c_double(); _lib.check(_lib.lib.rq_operator_time(op._h, 5|0x100, 3, 0, C.byref(ms))); print('factor graph ms', ms.value)
prof('B after graph', fh)
comp=sys.argv[2] if len(sys.argv)>2 else None
if comp:
    PI=rq.baseline_config(comp, device=True); prof('D after companion assembly', fh)
    oI=rq.nested_dissection_order(PI); opI=rq.build_operator(PI,-0.5,oI); prof('E after companion operator', fh)
    _lib.check(_lib.lib.rq_operator_time(opI._h, 5|0x100, 3, 0, C.byref(ms))); prof('F after companion factor', fh)
    del opI; prof('G after companion op del', fh)
    del PI; prof('H after companion pencil del', fh)
pairs=op.solve_quadratic(100 if 'cfg4' in cfg else 20, eps=1e-10, raise_partial=False)
prof('C after eigs', fh)

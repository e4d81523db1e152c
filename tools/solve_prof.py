"""Triangular-solve timing per config (development aid): device ms of one
solve (fwd+bwd sweeps) warm and with an L2 scrub, and the GB/s it implies."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import paper_2112_14064_b200 as rq
from paper_2112_14064_b200 import _lib
for cfg in sys.argv[1:]:
    P = rq.baseline_config(cfg)
    op = rq.build_operator(P, -0.5)
    from paper_2112_14064_b200 import sparsela as sl
    st = sl.Ordering(P.n, P.box, P.elems).stats
    def t(what, iters):
        ms = C.c_double()
        _lib.check(_lib.lib.rq_operator_time(op._h, what, iters, 0, C.byref(ms)))
        return ms.value
    t(1, 5)
    warm, cold = t(1, 50), t(1 | 0x100, 20)
    print(f"{cfg}: solve warm {warm*1e3:.1f} us cold {cold*1e3:.1f} us  bytes {st['trisolve_bytes']:.3g} "
          f"-> {st['trisolve_bytes']/cold/1e6:.0f} GB/s cold", flush=True)

"""Distance of the returned eigenvalues to the closed-form cluster value
(development aid): cfg, block, seeds."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_14064_b200 as rq  # noqa: E402

CL = -0.03 + 1j * np.sqrt(0.9991)
name, block = sys.argv[1], int(sys.argv[2])
P = rq.baseline_config(name)
op = rq.build_operator(P, -0.5)
for seed in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    pairs = op.solve_quadratic(100 if name.startswith("cfg4") else 50, eps=1e-10, max_restarts=400, block=block,
                               seed=seed, raise_partial=False)
    lam = np.array([p.lam for p in pairs])
    d = np.minimum(np.abs(lam - CL), np.abs(lam - np.conj(CL)))
    print(f"{name} block {block} seed {seed}: max dist {d.max():.2e} median {np.median(d):.2e} "
          f"resid max {max(p.residual for p in pairs):.2e} cycles {op.last_info['restarts']}", flush=True)

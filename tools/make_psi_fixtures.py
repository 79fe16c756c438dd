"""Converged weights of the benchmark configurations, as committed fixtures.

The bench workload (BASELINE.json metric: cells/s "at psi converged for the
config's first Newton solve") needs the weights of a cold-start Newton solve.
They are computed ONCE on a B200 by the device solver (robust restriction,
eps_vol = 1%) and committed as float32 (tests/golden/psi_<cfg>.npz); every
consumer -- bench.py's GPU arm, its reference (CPU) arm, the parity census
and the full-size parity tests -- reads float64(psi_f32), so both arms time
bit-identical inputs and the reference arm never loads the CUDA library.
(float32 rounding moves psi by <= 6e-8 relative: volumes by ~1e-7, far
inside the 1% convergence tolerance.)

usage (GPU box): python tools/make_psi_fixtures.py C4 C2 ... [--out DIR]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    import torch

    from paper_2601_05765_b200 import geom, scenes, solver

    os.makedirs(a.out, exist_ok=True)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    for cfg in a.configs:
        sc = scenes.make(cfg)
        res = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"), dom)
        psi = res.psi.cpu().numpy().astype(np.float32)
        meta = {k: (v if isinstance(v, (int, float, str)) else str(v)) for k, v in res.stats.items()}
        np.savez_compressed(os.path.join(a.out, f"psi_{cfg}.npz"), psi=psi, n=sc.n,
                            meta=json.dumps({"config": cfg, "solver": "device pf_newton_solve, robust restriction, "
                                             "cold start, eps_vol 0.01", **meta}))
        print(cfg, sc.n, meta, flush=True)


if __name__ == "__main__":
    main()

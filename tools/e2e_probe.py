"""Timeline of the host-array drop-in (pf_batch_evaluate_host) on a config at
its converged weights: per call wall time, and with PF_HOST_TRACE=1 the
per-range kernels / copy / scatter completion times (dev tool).
usage: python tools/e2e_probe.py [CONFIG] [CHUNKS ...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2601_05765_b200 import _kernels, geom, laguerre, scenes

    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    chunks = [int(k) for k in sys.argv[2:]] or [16]
    sc = scenes.make(cfg)
    psi = np.load(os.path.join(ROOT, "tests", "golden", f"psi_{cfg}.npz"))["psi"].astype(np.float64)
    dpk = laguerre.domain_pack(geom.box_domain([0, 0, 0], [1, 1, 1]))
    n, smf = sc.n, 32
    outs = [np.zeros(n, np.int64), np.zeros(n), np.zeros(n), np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n),
            np.zeros(n, np.int64), np.zeros((n, smf), np.int64), np.zeros((n, smf)), np.zeros((n, smf)),
            np.zeros((n, smf, 3)), np.zeros((n, smf, 3))]
    gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
    pts = np.ascontiguousarray(sc.pts)
    for K in chunks:
        os.environ["PF_E2E_CHUNKS"] = str(K)
        ts = []
        for it in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _kernels._batch_evaluate(pts, psi, *dpk.args(), *gargs, dpk.tol, -1.0, True, True, smf, *outs)
            ts.append(1e3 * (time.perf_counter() - t0))
        print(f"{cfg} K={K}: ms per call {[round(t, 1) for t in ts]}", flush=True)


if __name__ == "__main__":
    main()

"""Speed of the CPU baseline (oracle/potflow_oracle.c, the bit-identical C
restatement of the reference kernel) against the REAL numba reference
(_kernels._batch_evaluate), same inputs, same thread count, in the build
container (where /root/reference exists; the GPU box does not have it).
Writes profiles/port_vs_numba.json, which bench.py reports as
cpu_baseline.port_vs_numba.  usage: python tools/port_vs_numba.py [CONFIG]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    threads = os.cpu_count()
    os.environ.setdefault("NUMBA_NUM_THREADS", str(threads))
    from make_golden import import_reference

    geom_r, lag_r, kern_r = import_reference()
    import potflow

    potflow.set_threads(threads)
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import scenes

    sc = scenes.make(cfg)
    psi = np.load(os.path.join(ROOT, "tests", "golden", f"psi_{cfg}.npz"))["psi"].astype(np.float64)
    pts = np.ascontiguousarray(sc.pts)
    n, smf = len(pts), 32
    dom = geom_r.box_domain([0, 0, 0], [1, 1, 1]) if hasattr(geom_r, "box_domain") else None
    dp = lag_r.domain_pack(dom)

    def outs():
        return [np.zeros(n, np.int64), np.zeros(n), np.zeros(n), np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n),
                np.zeros(n, np.int64), np.zeros((n, smf), np.int64), np.zeros((n, smf)), np.zeros((n, smf)),
                np.zeros((n, smf, 3)), np.zeros((n, smf, 3))]

    res = {"config": cfg, "n": n, "threads": threads}
    # numba reference (JIT warm-up on a small slice first)
    g = lag_r.SpatialGrid(pts, dom)
    small = outs()
    kern_r._batch_evaluate(pts[:2000], psi[:2000], *dp.args(), *lag_r.SpatialGrid(pts[:2000], dom).kernel_args(),
                           dp.tol, lag_r._dpsi_max(psi[:2000]), True, True, smf, *[a[:2000] for a in small])
    o_ref = outs()
    t0 = time.perf_counter()
    g = lag_r.SpatialGrid(pts, dom)
    kern_r._batch_evaluate(pts, psi, *dp.args(), *g.kernel_args(), dp.tol, lag_r._dpsi_max(psi), True, True, smf,
                           *o_ref)
    res["numba_s"] = time.perf_counter() - t0
    # the C port, same workload and threads, grid build included
    o_port = outs()
    t0 = time.perf_counter()
    gp = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], dp.volume)
    O.batch_evaluate(pts, psi, *dp.args(), *gp.kernel_args(), dp.tol, O.dpsi_max(psi), True, True, smf, *o_port)
    res["port_s"] = time.perf_counter() - t0
    res["port_vs_numba"] = res["numba_s"] / res["port_s"]
    res["outputs_identical"] = bool(all(np.array_equal(a, b) for a, b in zip(o_ref, o_port)))
    res["numba_cells_per_s"] = n / res["numba_s"]
    res["port_cells_per_s"] = n / res["port_s"]
    out = os.path.join(ROOT, "profiles", "port_vs_numba.json" if cfg == "C4" else f"port_vs_numba_{cfg}.json")
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

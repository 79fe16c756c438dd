"""The HBM-bound kernels of the path on the bench workload (C4 at its
converged weights), inside a cudaProfilerStart/Stop range for
`ncu --profile-from-start off --metrics dram__bytes_read.sum,...`:
grid counting sort (pf_grid_build), 16 Jacobi-PCG iterations on the Newton
Hessian (pf_pcg), and the exact kNN of every site (pf_knn, k=16).
Prints the CUDA-event times as JSON (never a bench number under ncu)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2601_05765_b200 import _lib, geom, laguerre, restricted, scenes, solver

    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    sc = scenes.make(cfg)
    psi = np.load(os.path.join(ROOT, "tests", "golden", f"psi_{cfg}.npz"))["psi"].astype(np.float64)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    L = solver._bind()
    c = _lib.ctx()
    laguerre.upload_domain(c, *dpk.args(), dpk.tol)
    n, smf = sc.n, 32
    pts = torch.as_tensor(sc.pts, device="cuda")
    pg = torch.as_tensor(psi, device="cuda")
    s = _lib.stream_ptr()
    f8, i4 = dict(dtype=torch.float64, device="cuda"), dict(dtype=torch.int32, device="cuda")
    # lean evaluation -> Hessian (untimed set-up)
    _lib.check(L.pf_grid_build(c, n, _lib.ptr(pts), _lib.ptr(pg), 0.0, s), "pf_grid_build")
    vol, ksur = torch.empty(n, **f8), torch.empty(n, **f8)
    fcount, ftag, farea = torch.empty(n, **i4), torch.empty((n, smf), **i4), torch.empty((n, smf), **f8)
    cent = torch.empty((n, 3), **f8)
    flags = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(L.pf_evaluate_lean(c, n, _lib.ptr(pts), _lib.ptr(pg), 1, smf, _lib.ptr(vol), _lib.ptr(ksur),
                                  _lib.ptr(fcount), _lib.ptr(ftag), _lib.ptr(farea), _lib.ptr(cent),
                                  _lib.ptr(flags), s), "pf_evaluate_lean")
    hcnt, hcol = torch.empty(n, **i4), torch.empty((n, smf), **i4)
    hval, diag = torch.empty((n, smf), **f8), torch.empty(n, **f8)
    _lib.check(L.pf_newton_hessian(n, smf, _lib.ptr(pts), _lib.ptr(pg), _lib.ptr(fcount), _lib.ptr(ftag),
                                   _lib.ptr(farea), _lib.ptr(ksur), float(1e-12 * dom.diagonal() ** 2),
                                   _lib.ptr(hcnt), _lib.ptr(hcol), _lib.ptr(hval), _lib.ptr(diag), s),
               "pf_newton_hessian")
    b = torch.rand(n, generator=torch.Generator(device="cuda").manual_seed(1), **f8)
    x = torch.empty(n, **f8)
    q = pts.clone()
    knn = torch.empty((n, 16), dtype=torch.int64, device="cuda")
    L.pf_pcg(n, smf, _lib.ptr(hcnt), _lib.ptr(hcol), _lib.ptr(hval), _lib.ptr(diag), _lib.ptr(b), _lib.ptr(x),
             0.0, 4, s)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.profiler.start()
    ev[0].record()
    _lib.check(L.pf_grid_build(c, n, _lib.ptr(pts), _lib.ptr(pg), 0.0, s), "pf_grid_build")
    ev[1].record()
    it = L.pf_pcg(n, smf, _lib.ptr(hcnt), _lib.ptr(hcol), _lib.ptr(hval), _lib.ptr(diag), _lib.ptr(b),
                  _lib.ptr(x), 0.0, 16, s)
    ev[2].record()
    got = L.pf_knn(c, n, _lib.ptr(pts), n, _lib.ptr(q), 16, _lib.ptr(knn), 0, s)
    ev[3].record()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    nnz = int(hcnt.sum())
    print(json.dumps({"n": n, "nnz": nnz, "pcg_iterations": it, "knn_k": got,
                      "grid_ms": ev[0].elapsed_time(ev[1]), "pcg_ms": ev[1].elapsed_time(ev[2]),
                      "knn_ms": ev[2].elapsed_time(ev[3])}))


if __name__ == "__main__":
    main()

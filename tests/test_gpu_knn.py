"""Exact k-nearest sites (pf_knn, the _knn drop-in's kernel) at BASELINE
sizes against a numpy brute force with the kernel's own d^2 arithmetic and the
reference's (d^2, j) order (_kernels.py:1562-1620): the sites of C2 (97k,
lattice) and C5 (1M, two densities) as queries, plus random points anywhere in
the box (empty regions included), k = 1, 7, 16, 40."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _brute(pts, q, k):
    out = np.empty((len(q), k), np.int64)
    idx = np.arange(len(pts))
    for a, p in enumerate(q):
        d2 = ((pts[:, 0] - p[0]) ** 2 + (pts[:, 1] - p[1]) ** 2) + (pts[:, 2] - p[2]) ** 2
        kth = np.partition(d2, k - 1)[k - 1]
        part = idx[d2 <= kth]  # every tie of the k-th distance
        o = np.lexsort((part, d2[part]))[:k]
        out[a] = part[o]
    return out


@pytest.mark.parametrize("cfg", ["C2", "C5"])
def test_knn_exact_at_size(cfg):
    from paper_2601_05765_b200 import _kernels, geom, laguerre, scenes

    sc = scenes.make(cfg)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    rng = np.random.default_rng(3)
    q_sites = sc.pts[rng.choice(sc.n, 600, replace=False)]
    q_rand = rng.random((400, 3))
    for k in (1, 7, 16, 40):
        for q in (q_sites, q_rand):
            got = laguerre.knn_batch(sc.pts, q, k, dom)
            got = got.cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
            want = _brute(sc.pts, q, k)
            assert np.array_equal(got, want), (cfg, k)

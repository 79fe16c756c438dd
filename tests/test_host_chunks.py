"""Index ranges of the host-array drop-in (_kernels._chunk_bounds): they
partition [0, n) in order, the trailing ranges shrink, and the range id of a
cell index (torch.bucketize, as the drop-in assigns cells) is the range holding
it.  CPU only."""
import numpy as np
import pytest


@pytest.mark.parametrize("n,K", [(0, 1), (1, 16), (5, 16), (100, 16), (1940519, 16), (97336, 8), (1000, 4)])
def test_chunk_bounds_partition(n, K):
    import torch

    from paper_2601_05765_b200._kernels import _chunk_bounds

    K = max(1, min(K, max(n, 1)))
    b = _chunk_bounds(n, K)
    assert len(b) == K + 1 and b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
    if K >= 6 and n >= 1000:
        sz = np.diff(b)
        assert sz[-1] < sz.max() / 4
    if n:
        idx = torch.arange(n)
        rid = torch.bucketize(idx, torch.as_tensor(b[1:-1]), right=True).numpy()
        for k in range(K):
            assert np.all(rid[b[k]:b[k + 1]] == k)

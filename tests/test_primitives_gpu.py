"""GPU: the radix sort and scan primitives behind K2/K5 (stability is what
gives the reference's (count desc, row asc) tie-break)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bits", [(1, 8), (5, 3), (2047, 11), (2048, 8), (4096, 16), (4097, 32),
                                    (100_003, 20), (1 << 20, 32), (3_000_001, 28),
                                    (12_345_678, 24)])
def test_radix_sort_pairs_stable(cuda_ctx, n, bits):
    import torch

    from paper_2201_10095_b200 import _lib
    from paper_2201_10095_b200.runtime import ptr

    rng = np.random.default_rng(n)
    hi = (1 << bits) - 1
    keys = rng.integers(0, min(hi, 1 << 12) + 1 if n > 4096 else hi + 1, n, dtype=np.uint64)
    keys = (keys * (hi // max(1, keys.max() or 1))).astype(np.uint32) & np.uint32(hi)
    vals = np.arange(n, dtype=np.uint32)
    dk = torch.from_numpy(keys.view(np.int32)).cuda()
    dv = torch.from_numpy(vals.view(np.int32)).cuda()
    _lib.check(_lib.lib().rs_radix_sort_pairs(cuda_ctx.h, ptr(dk), ptr(dv), C.c_uint64(n), bits))
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(dk.cpu().numpy().view(np.uint32), keys[order])
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), vals[order])


def test_radix_sort_pairs_skewed(cuda_ctx):
    """Zipf-skewed keys (most tiles hold one digit): look-back and stability."""
    import torch

    from paper_2201_10095_b200 import _lib
    from paper_2201_10095_b200.runtime import ptr

    rng = np.random.default_rng(7)
    n = 2_000_003
    keys = np.minimum(rng.zipf(1.3, n) - 1, (1 << 27) - 1).astype(np.uint32)
    keys[: n // 3] = 5  # a long run of one key
    vals = np.arange(n, dtype=np.uint32)
    dk = torch.from_numpy(keys.view(np.int32)).cuda()
    dv = torch.from_numpy(vals.view(np.int32)).cuda()
    _lib.check(_lib.lib().rs_radix_sort_pairs(cuda_ctx.h, ptr(dk), ptr(dv), C.c_uint64(n), 27))
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(dk.cpu().numpy().view(np.uint32), keys[order])
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), vals[order])

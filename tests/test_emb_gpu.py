"""GPU parity: the tiered EmbeddingBag (K4 forward, K5 backward + optimizer).

Oracle: oracle.c's or_emb_forward / or_emb_backward (paper semantics; parity
unpinned at the reference boundary).  Forward is bit-exact
(same fp32 accumulation order); the backward is checked to 1e-5 relative
(BASELINE.json north_star tolerance) and for bitwise run-to-run determinism.
"""
import numpy as np
import pytest

import paper_2201_10095_b200 as sp
from paper_2201_10095_b200.types import PlanEntry, TableSpec

pytestmark = pytest.mark.gpu

SEED = 99
SCALE = 0.5


def _setup(coracle, dims, Hs, hbm_frac, B, max_len, rng, zipf=False):
    import torch

    specs = [TableSpec(10 + t, H, H, d, 4) for t, (d, H) in enumerate(zip(dims, Hs))]
    remaps = []
    for s, f in zip(specs, hbm_frac):
        counts = rng.integers(0, 4, s.hash_size)
        rbr = sorted(np.nonzero(counts)[0].tolist(), key=lambda r: (-counts[r], r))
        st = sp.FeatureStats(s.table_id, 1.0, 1.0, len(rbr), 0, np.zeros(101, np.uint64),
                             np.zeros(len(rbr)), np.array(rbr, np.uint32))
        remaps.append(sp.build_remap(PlanEntry(s.table_id, 0, 0, int(f * s.hash_size)), st, s))
    T = len(specs)
    lens = rng.integers(0, max_len + 1, T * B)
    lens[rng.random(T * B) < 0.1] = 0  # absent features pool to zero
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    idx = []
    for i, L in enumerate(lens):
        H = Hs[i // B]
        if zipf:
            idx.append(np.minimum(rng.zipf(1.2, L) - 1, H - 1))
        else:
            idx.append(rng.integers(0, H, L))
    idx = np.concatenate(idx).astype(np.uint32) if len(idx) else np.zeros(0, np.uint32)
    d_off = torch.from_numpy(offsets.view(np.int32)).cuda()
    d_idx = torch.from_numpy(idx.view(np.int32)).cuda()
    Ws = [coracle.init_table(SEED, s.table_id, s.hash_size, s.dim, SCALE) for s in specs]
    return specs, remaps, offsets, idx, d_off, d_idx, Ws


CASES = [
    ([64, 128, 32], [1000, 3000, 257], [0.5, 0.2, 1.0], 256, 30),
    ([256, 96, 4], [500, 800, 64], [0.0, 0.7, 0.3], 100, 12),
    ([64], [50], [0.4], 1024, 40),  # heavy duplicates: long row segments cross chunks
    ([64, 128], [4, 3], [0.5, 0.34], 2048, 30),  # segments of ~15K: cross superchunks
]


@pytest.mark.parametrize("case", CASES)
def test_forward_bit_exact_and_hit_counts(cuda_ctx, coracle, case):
    import torch

    dims, Hs, frac, B, ml = case
    rng = np.random.default_rng(1)
    specs, remaps, offsets, idx, d_off, d_idx, Ws = _setup(coracle, dims, Hs, frac, B, ml, rng)
    op = sp.TieredEmbeddingBag(specs, remaps, B, max(1, idx.size), "sgd", ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    hits = torch.zeros(2 * len(specs), dtype=torch.int64, device="cuda")
    out = op.forward(d_off, d_idx, B, hits=hits)
    torch.cuda.synchronize()
    want = coracle.emb_forward(B, dims, offsets.astype(np.uint64), idx, Ws)
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    h = hits.cpu().numpy()
    for t, r in enumerate(remaps):
        seg = idx[offsets[t * B]:offsets[(t + 1) * B]]
        fast = int((r.entries[seg] >= 0).sum())
        assert h[2 * t] == fast and h[2 * t + 1] == seg.size - fast
    # tier placement: every row reads back as its deterministic init
    for t, s in enumerate(specs):
        rows = np.arange(s.hash_size, dtype=np.uint32)
        w, _ = op.read_rows(t, rows)
        assert np.array_equal(w, Ws[t])
    op.close()


@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
@pytest.mark.parametrize("case", CASES)
def test_backward_matches_oracle(cuda_ctx, coracle, case, opt):
    import torch

    dims, Hs, frac, B, ml = case
    rng = np.random.default_rng(2)
    specs, remaps, offsets, idx, d_off, d_idx, Ws = _setup(coracle, dims, Hs, frac, B, ml, rng,
                                                           zipf=True)
    op = sp.TieredEmbeddingBag(specs, remaps, B, max(1, idx.size), opt, eps=1e-8, ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    grad = rng.standard_normal((B, sum(dims))).astype(np.float32)
    lr = 0.05
    for _ in range(2):  # two steps: the second sees updated weights and momentum
        op.backward(d_off, d_idx, torch.from_numpy(grad).cuda(), B, lr)
    torch.cuda.synchronize()
    mom = [np.zeros(s.hash_size, np.float32) for s in specs]
    for _ in range(2):
        coracle.emb_backward(B, dims, offsets.astype(np.uint64), idx, grad, Ws, mom,
                             0 if opt == "sgd" else 1, lr, 1e-8,
                             remaps=[(r.entries, r.hbm_rows) for r in remaps])
    for t, s in enumerate(specs):
        w, m = op.read_rows(t, np.arange(s.hash_size, dtype=np.uint32))
        # north_star tolerance: 1e-5 relative ...
        np.testing.assert_allclose(w, Ws[t], rtol=1e-5, atol=1e-6)
        # ... and in fact bit-exact: the oracle restates the kernel's fixed
        # reduction order (oracle.h or_emb_backward)
        assert np.array_equal(w.view(np.uint32), Ws[t].view(np.uint32))
        if opt != "sgd":
            assert np.array_equal(m.view(np.uint32), mom[t].view(np.uint32))
    op.close()


def test_backward_deterministic(cuda_ctx, coracle):
    import torch

    dims, Hs, frac, B, ml = CASES[0]
    outs = []
    for _ in range(2):
        rng = np.random.default_rng(3)
        specs, remaps, offsets, idx, d_off, d_idx, Ws = _setup(coracle, dims, Hs, frac, B, ml, rng,
                                                               zipf=True)
        op = sp.TieredEmbeddingBag(specs, remaps, B, idx.size, "rowwise_adagrad", ctx=cuda_ctx)
        op.init_weights(SEED, SCALE)
        g = torch.from_numpy(rng.standard_normal((B, sum(dims))).astype(np.float32)).cuda()
        for _ in range(3):
            y = op.forward(d_off, d_idx, B)
            op.backward(d_off, d_idx, g + 0.01 * y, B, 0.1)
        torch.cuda.synchronize()
        outs.append([op.read_rows(t, np.arange(s.hash_size, dtype=np.uint32)) for t, s in
                     enumerate(specs)])
        op.close()
    for (wa, ma), (wb, mb) in zip(*outs):
        assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))
        assert np.array_equal(ma.view(np.uint32), mb.view(np.uint32))


def _train(cuda_ctx, coracle, cached, steps=5, nslots=4096, depth=1):
    """Fwd+bwd over distinct batches; with `cached`, batch k+depth is
    prefetched (slow rows staged in HBM) while batch k runs."""
    import torch

    dims, Hs, frac, B, ml = ([64, 128, 32], [300, 500, 2000], [0.3, 0.1, 0.5], 128, 12)
    rng = np.random.default_rng(11)
    specs, remaps, _, _, _, _, _ = _setup(coracle, dims, Hs, frac, B, ml, rng)
    batches = []
    for k in range(steps):
        r2 = np.random.default_rng(100 + k)
        lens = r2.integers(0, ml + 1, len(dims) * B)
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
        idx = np.concatenate([np.minimum(r2.zipf(1.3, L) - 1, Hs[i // B] - 1)
                              for i, L in enumerate(lens)]).astype(np.uint32)
        batches.append((torch.from_numpy(off.view(np.int32)).cuda(),
                        torch.from_numpy(idx.view(np.int32)).cuda(), idx.size))
    op = sp.TieredEmbeddingBag(specs, remaps, B, max(b[2] for b in batches), "rowwise_adagrad",
                               ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    if cached:
        op.enable_uvm_cache(nslots)
        for k in range(min(depth, steps)):
            op.prefetch(batches[k][0], batches[k][1], B)
    outs = []
    for k in range(steps):
        off, idx, _ = batches[k]
        y = op.forward(off, idx, B)
        if cached and k + depth < steps:
            op.prefetch(batches[k + depth][0], batches[k + depth][1], B)
        outs.append(y.clone())
        op.backward(off, idx, y * 0.5 + 0.01, B, 0.05)
    torch.cuda.synchronize()
    rows = [op.read_rows(t, np.arange(s.hash_size, dtype=np.uint32)) for t, s in enumerate(specs)]
    op.close()
    return outs, rows


def test_uvm_cache_bit_identical_to_zero_copy(cuda_ctx, coracle):
    """Slow rows staged in HBM with side-stream prefetch/write-back (one batch
    ahead) give exactly the zero-copy results, incl. rows shared by
    consecutive batches and slot reuse under a small cache."""
    ref_out, ref_rows = _train(cuda_ctx, coracle, cached=False)
    for nslots in (4096, 1800):
        out, rows = _train(cuda_ctx, coracle, cached=True, nslots=nslots)
        for a, b in zip(out, ref_out):
            assert torch_equal(a, b)
        for (wa, ma), (wb, mb) in zip(rows, ref_rows):
            assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))
            assert np.array_equal(ma.view(np.uint32), mb.view(np.uint32))


@pytest.mark.parametrize("nslots", [4096, 2600])
def test_uvm_cache_two_batches_ahead_bit_identical(cuda_ctx, coracle, nslots):
    """Staging two batches ahead (the bench's pipeline: four generations live —
    one awaiting eviction, the current one, two staged) gives exactly the
    zero-copy results."""
    ref_out, ref_rows = _train(cuda_ctx, coracle, cached=False, steps=7)
    out, rows = _train(cuda_ctx, coracle, cached=True, steps=7, nslots=nslots, depth=2)
    for a, b in zip(out, ref_out):
        assert torch_equal(a, b)
    for (wa, ma), (wb, mb) in zip(rows, ref_rows):
        assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))
        assert np.array_equal(ma.view(np.uint32), mb.view(np.uint32))


def torch_equal(a, b):
    import torch

    return bool(torch.equal(a.view(torch.int32), b.view(torch.int32)))


def test_uvm_cache_errors(cuda_ctx, coracle):
    """Out of staging slots: the batch is refused BEFORE its forward runs (no
    kernel touches an unfilled slot), flush() empties the cache and clears the
    error, and the operator then runs zero-copy with the oracle's results."""
    import torch

    rng = np.random.default_rng(5)
    specs, remaps, offsets, idx, d_off, d_idx, Ws = _setup(coracle, [64], [1000], [0.0], 64, 10, rng)
    op = sp.TieredEmbeddingBag(specs, remaps, 64, idx.size, "sgd", ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    with pytest.raises(sp.InvalidArgument):  # prefetch needs the cache
        op.prefetch(d_off, d_idx, 64)
    op.enable_uvm_cache(4)  # far fewer slots than slow rows in the batch
    op.prefetch(d_off, d_idx, 64)
    op.prefetch(d_off, d_idx, 64)  # the next batch and the one after: two live
    with pytest.raises(sp.InvalidArgument):  # a third would be two batches ahead
        op.prefetch(d_off, d_idx, 64)
    with pytest.raises(sp.InvalidArgument):  # out of slots: refused before the forward
        op.forward(d_off, d_idx, 64)
    with pytest.raises(sp.InvalidArgument):  # flush reports it once, then the cache is clean
        op.flush()
    op.flush()
    y = op.forward(d_off, d_idx, 64)  # zero-copy again
    want = coracle.emb_forward(64, [64], offsets.astype(np.uint64), idx, Ws)
    assert np.array_equal(y.cpu().numpy(), want)
    torch.cuda.synchronize()
    op.close()


def test_operator_rejects_bad_inputs(cuda_ctx):
    spec = TableSpec(0, 10, 10, 6, 4)  # dim not a multiple of 4
    r = sp.RemapTable(0, 10, 10, 0, np.arange(10, dtype=np.int32))
    with pytest.raises(sp.InvalidArgument):
        sp.TieredEmbeddingBag([spec], [r], 4, 16, ctx=cuda_ctx)
    spec = TableSpec(0, 10, 10, 8, 4)
    bad = sp.RemapTable(0, 10, 5, 0, np.arange(10, dtype=np.int32))  # entry beyond hbm_rows
    with pytest.raises(sp.InvalidArgument):
        sp.TieredEmbeddingBag([spec], [bad], 4, 16, ctx=cuda_ctx)


def test_out_of_range_index_is_reported(cuda_ctx, coracle):
    """An index >= hash_size never reads out of bounds; the next backward
    raises InvalidArgument (the reference rejects hashed ids outside H)."""
    import torch

    rng = np.random.default_rng(8)
    specs, remaps, offsets, idx, d_off, d_idx, _ = _setup(coracle, [16], [100], [0.5], 8, 4, rng)
    op = sp.TieredEmbeddingBag(specs, remaps, 8, max(1, idx.size), "sgd", ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    bad = d_idx.clone()
    if bad.numel():
        bad[0] = 100  # == hash_size
    y = op.forward(d_off, bad, 8)
    with pytest.raises(sp.InvalidArgument):
        op.backward(d_off, bad, y, 8, 0.1)
    # the error is consumed: a clean batch runs again
    y = op.forward(d_off, d_idx, 8)
    op.backward(d_off, d_idx, y, 8, 0.1)
    torch.cuda.synchronize()
    op.close()


def test_backward_rejects_bad_batches_without_touching_weights(cuda_ctx, coracle):
    """The backward validates its batch on the device (bwd_plan_kernel) and
    raises the documented InvalidArgument; an empty plan means no row moves.
    A batch the last forward did not see goes through the stand-alone keygen,
    whose index errors empty the plan too."""
    import torch

    rng = np.random.default_rng(21)
    specs, remaps, offsets, idx, d_off, d_idx, _ = _setup(coracle, [16, 32], [100, 60], [0.5, 0.3], 16, 6, rng)
    op = sp.TieredEmbeddingBag(specs, remaps, 16, max(1, idx.size), "rowwise_adagrad", ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    rows = [np.arange(s.hash_size, dtype=np.uint32) for s in specs]

    def snapshot():
        torch.cuda.synchronize()
        return [op.read_rows(t, r) for t, r in enumerate(rows)]

    def same(a, b):
        return all(np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]) for x, y in zip(a, b))

    y = op.forward(d_off, d_idx, 16)
    before = snapshot()
    bad_start = d_off.clone()
    bad_start[0] = 1
    bad_order = d_off.clone()
    k = int(np.nonzero(np.diff(offsets) > 0)[0][0]) + 1  # an offset that can be lowered
    bad_order[k] = int(offsets[k - 1]) - 1 if offsets[k - 1] > 0 else int(offsets[k + 1]) + 5
    bad_bound = d_off.clone()
    bad_bound[16] = int(offsets[32]) + 1  # table 1 starts after table 2
    too_many = d_off.clone()
    too_many[-1] = idx.size + 1
    bad_idx = d_idx.clone()
    bad_idx[0] = 100  # == hash_size of table 0
    cases = [(bad_start, d_idx, "offsets must start at 0"),
             (bad_order, d_idx, "non-decreasing"),
             (bad_bound, d_idx, "non-decreasing"),
             (too_many, d_idx, "more lookups than max_lookups"),
             (d_off.clone(), bad_idx, "outside its table's hash_size")]
    for o, i, msg in cases:
        with pytest.raises(sp.InvalidArgument, match=msg):
            op.backward(o, i, y, 16, 0.1)
        assert same(snapshot(), before), msg
    # the operator is clean afterwards
    y = op.forward(d_off, d_idx, 16)
    op.backward(d_off, d_idx, y, 16, 0.1)
    assert not same(snapshot(), before)
    op.close()


@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
def test_backward_tree_edges(cuda_ctx, coracle, opt):
    """Segment lengths on every edge of the reduction tree (oracle.h): 1, 31,
    32 (one piece), 33 (two pieces), 2048 (64 pieces = one group), 2049 (two
    groups), 4160 — bit-exact vs the oracle, both tiers."""
    import torch

    counts = [1, 31, 32, 33, 2048, 2049, 4160, 5]
    H = len(counts)
    rng = np.random.default_rng(21)
    idx = np.repeat(np.arange(H, dtype=np.uint32), counts)
    rng.shuffle(idx)
    B = idx.size  # one lookup per bag
    offsets = np.arange(B + 1, dtype=np.uint32)
    spec = TableSpec(3, H, H, 64, 4)
    st = sp.FeatureStats(3, 1.0, 1.0, H, B, np.zeros(101, np.uint64), np.zeros(H),
                         np.arange(H, dtype=np.uint32))
    remap = sp.build_remap(PlanEntry(3, 0, 0, 4), st, spec)  # rows 0-3 fast, 4-7 slow
    op = sp.TieredEmbeddingBag([spec], [remap], B, B, opt, eps=1e-8, ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    grad = rng.standard_normal((B, 64)).astype(np.float32)
    d_off = torch.from_numpy(offsets.view(np.int32)).cuda()
    d_idx = torch.from_numpy(idx.view(np.int32)).cuda()
    op.backward(d_off, d_idx, torch.from_numpy(grad).cuda(), B, 0.05)
    torch.cuda.synchronize()
    W = [coracle.init_table(SEED, 3, H, 64, SCALE)]
    mom = [np.zeros(H, np.float32)]
    coracle.emb_backward(B, [64], offsets.astype(np.uint64), idx, grad, W, mom,
                         0 if opt == "sgd" else 1, 0.05, 1e-8,
                         remaps=[(remap.entries, remap.hbm_rows)])
    w, m = op.read_rows(0, np.arange(H, dtype=np.uint32))
    assert np.array_equal(w.view(np.uint32), W[0].view(np.uint32))
    if opt != "sgd":
        assert np.array_equal(m.view(np.uint32), mom[0].view(np.uint32))
    op.close()

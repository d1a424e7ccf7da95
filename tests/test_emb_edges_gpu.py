"""Edge cases of the tiered EmbeddingBag (the reference tests empty and
degenerate inputs at its own boundaries; the operator has none, so these
follow the paper's semantics: an empty bag pools to 0, and a
batch without lookups updates nothing):

* every bag empty — the forward writes zeros, the backward leaves every row
  and state bit-identical, in the zero-copy and in the staged mode;
* one bag, one table of one row, both optimizers;
* the reduction-tree edges (segments of 1, 31-33, 2048-2049, 4160 lookups)
  on fp16 rows, against the fp64 oracle with one fp16 ulp of slack;
* a lookup batch larger than one launch's persistent grid (every warp
  claims many chunks).
"""
import numpy as np
import pytest

import paper_2201_10095_b200 as sp
from oracle import emb64
from paper_2201_10095_b200.types import PlanEntry, TableSpec

pytestmark = pytest.mark.gpu

SEED, SCALE = 5, 0.5


def _remap(spec, hbm):
    H = spec.hash_size
    st = sp.FeatureStats(spec.table_id, 1.0, 1.0, H, 0, np.zeros(101, np.uint64), np.zeros(H),
                         np.arange(H, dtype=np.uint32))
    return sp.build_remap(PlanEntry(spec.table_id, 0, 0, hbm), st, spec)


@pytest.mark.parametrize("staged", [False, True])
def test_all_bags_empty(cuda_ctx, coracle, staged):
    import torch

    specs = [TableSpec(1, 300, 300, 64, 4), TableSpec(2, 70, 70, 128, 2), TableSpec(3, 9, 9, 8, 4)]
    remaps = [_remap(s, s.hash_size // 2) for s in specs]
    B = 777
    op = sp.TieredEmbeddingBag(specs, remaps, B, 16, "rowwise_adagrad", ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    before = [op.read_rows(t, np.arange(s.hash_size, dtype=np.uint32)) for t, s in enumerate(specs)]
    off = torch.zeros(len(specs) * B + 1, dtype=torch.int32, device="cuda")
    idx = torch.zeros(1, dtype=torch.int32, device="cuda")
    if staged:
        op.enable_uvm_cache(1024)
        op.prefetch(off, idx, B)
    y = op.forward(off, idx, B)
    assert not y.any()
    y.fill_(1.0)
    op.backward(off, idx, y, B, 0.5)
    if staged:
        op.flush()
    for t, s in enumerate(specs):
        w, m = op.read_rows(t, np.arange(s.hash_size, dtype=np.uint32))
        assert np.array_equal(w.view(np.uint32), before[t][0].view(np.uint32))
        assert np.array_equal(m.view(np.uint32), before[t][1].view(np.uint32))
    op.close()


@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
def test_one_row_one_bag(cuda_ctx, coracle, opt):
    import torch

    spec = TableSpec(4, 1, 1, 4, 4)
    op = sp.TieredEmbeddingBag([spec], [_remap(spec, 1)], 1, 3, opt, eps=1e-8, ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    off = torch.tensor([0, 3], dtype=torch.int32, device="cuda")
    idx = torch.zeros(3, dtype=torch.int32, device="cuda")
    y = op.forward(off, idx, 1)
    W = coracle.init_table(SEED, 4, 1, 4, SCALE)
    want, wabs = emb64.forward(1, [4], np.array([0, 3], np.uint64), np.zeros(3, np.uint32), [W])
    emb64.check(y.cpu().numpy(), want, emb64.RTOL * wabs + 1e-30, "forward")
    op.backward(off, idx, y, 1, 0.25)
    rows, g, ga = emb64.row_grads(1, [4], np.array([0, 3], np.uint64), np.zeros(3, np.uint32),
                                  y.cpu().numpy(), 0)
    wn, mn, wb, mb = emb64.update(W[rows], np.zeros(1, np.float32), g, ga, opt, 0.25, 1e-8)
    gw, gm = op.read_rows(0, rows)
    emb64.check(gw, wn, wb, "row")
    if opt != "sgd":
        emb64.check(gm, mn, mb, "state")
    op.close()


def test_tree_edges_fp16(cuda_ctx, coracle):
    import torch

    counts = [1, 31, 32, 33, 2048, 2049, 4160, 5]
    H = len(counts)
    rng = np.random.default_rng(3)
    idx = np.repeat(np.arange(H, dtype=np.uint32), counts)
    rng.shuffle(idx)
    B = idx.size
    off = np.arange(B + 1, dtype=np.uint32)
    spec = TableSpec(6, H, H, 128, 2)
    op = sp.TieredEmbeddingBag([spec], [_remap(spec, 4)], B, B, "rowwise_adagrad", eps=1e-8, ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    grad = (rng.standard_normal((B, 128)) * 0.01).astype(np.float32)
    d_off = torch.from_numpy(off.view(np.int32)).cuda()
    d_idx = torch.from_numpy(idx.view(np.int32)).cuda()
    op.backward(d_off, d_idx, torch.from_numpy(grad).cuda(), B, 0.05)
    torch.cuda.synchronize()
    W = coracle.init_table(SEED, 6, H, 128, SCALE).astype(np.float16).astype(np.float32)
    rows, g, ga = emb64.row_grads(B, [128], off.astype(np.uint64), idx, grad, 0)
    wn, mn, wb, mb = emb64.update(W[rows], np.zeros(rows.size, np.float32), g, ga, "rowwise_adagrad", 0.05, 1e-8)
    wb = wb + np.spacing(np.abs(wn).astype(np.float16)).astype(np.float64)
    gw, gm = op.read_rows(0, rows)
    emb64.check(gw, wn, wb, "fp16 rows")
    emb64.check(gm, mn, mb, "state")
    op.close()


def test_many_chunks_per_warp(cuda_ctx, coracle):
    """A batch of 2^18 bags on one dim-4 table (G = 1: 32 bags per warp-
    iteration), far more bag-groups than the persistent forward grid has
    warps; forward bit-exact against the kernel-order oracle."""
    import torch

    spec = TableSpec(7, 1000, 1000, 4, 4)
    rng = np.random.default_rng(8)
    B = 1 << 18
    lens = rng.integers(0, 4, B)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    idx = rng.integers(0, 1000, int(off[-1])).astype(np.uint32)
    op = sp.TieredEmbeddingBag([spec], [_remap(spec, 600)], B, idx.size, "sgd", ctx=cuda_ctx)
    op.init_weights(SEED, SCALE)
    y = op.forward(torch.from_numpy(off.view(np.int32)).cuda(), torch.from_numpy(idx.view(np.int32)).cuda(), B)
    W = [coracle.init_table(SEED, 7, 1000, 4, SCALE)]
    want = coracle.emb_forward(B, [4], off.astype(np.uint64), idx, W)
    assert np.array_equal(y.cpu().numpy(), want)
    op.close()

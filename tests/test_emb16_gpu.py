"""fp16 tables and omit_unaccessed remaps through the tiered EmbeddingBag
(VERDICT r1 "Next round" 8: the reference TableSpec allows elem_bytes 2,
inc/types.hpp:31,50-52; RemapOptions.omit_unaccessed leaves never-profiled
slow rows without storage, inc/remap.hpp:43-48, core/src/remap.cpp:85-96).

Against the independent fp64 oracle (oracle/emb64.py):
* fp16 rows are the fp32 init rounded to nearest-even (numpy astype); the
  forward sums their exact widenings, so it must land within 1e-5 of the
  fp64 sum; an updated row is the fp64 update rounded once to fp16, so the
  bound adds one fp16 ulp of the result; the row-wise Adagrad state stays
  fp32 (1e-5).
* unbacked rows (an omit_unaccessed remap built from one batch, trained on
  another) pool as zero rows, take no update, read back as zeros, and are
  counted per table exactly as numpy counts them; backed rows are updated
  with the gradients of every lookup, as without the option.
Zero-copy and staged (pipelined) slow tier, both optimizers.
"""
import numpy as np
import pytest

import oracle
import paper_2201_10095_b200 as sp
from oracle import emb64
from paper_2201_10095_b200 import workload as wl
from paper_2201_10095_b200.types import PlanEntry, Trace

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")]

GEN_SEED = 20260809
INIT_SEED = 99


def _batch(specs, B, seed):
    R = oracle.Ref()
    tr = R.generate_trace([(w.table, (w.gen.zipf_exponent, w.gen.mean_pooling, w.gen.coverage,
                                      w.gen.pooling_law)) for w in specs], B, seed)
    off, idx = oracle.trace_to_csr(tr, [w.table.table_id for w in specs], B)
    trace = Trace([w.table for w in specs], B, tr.rec_sample, tr.rec_table, tr.rec_offset, tr.rec_len,
                  ids=tr.ids)
    R.free_trace(tr)
    return off, idx, trace


def _ulp16(x):
    return np.spacing(np.abs(x).astype(np.float16)).astype(np.float64)


def _run(ctx, coracle, specs, B, opt, staged, omit, lr=0.5):
    import torch

    T = len(specs)
    dims = [w.table.dim for w in specs]
    # plan from one batch, train on another (unseen rows appear)
    _, _, ptrace = _batch(specs, B, GEN_SEED)
    off, idx, _ = _batch(specs, B, GEN_SEED + 1)
    stats = sp.profile(ptrace, 1.0, 7, ctx=ctx)
    remaps = [sp.build_remap(PlanEntry(w.table.table_id, 0, 0, int(0.4 * st.distinct_rows_accessed)),
                             st, w.table, omit_unaccessed=omit, ctx=ctx) for w, st in zip(specs, stats)]
    op = sp.TieredEmbeddingBag([w.table for w in specs], remaps, B, max(1, idx.size), opt, eps=1e-8, ctx=ctx)
    op.init_weights(INIT_SEED, 0.1)
    d_off = torch.from_numpy(off.astype(np.uint32).view(np.int32)).cuda()
    d_idx = torch.from_numpy(idx.view(np.int32)).cuda()
    if staged:
        op.enable_uvm_cache(4 * idx.size + 1024)
        op.prefetch(d_off, d_idx, B)
    hits = torch.zeros(2 * T, dtype=torch.int64, device="cuda")
    y = op.forward(d_off, d_idx, B, hits=hits)
    op.backward(d_off, d_idx, y, B, lr)
    if staged:
        op.flush()
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    lk, nrows = op.unbacked()
    # oracle weights: storage-rounded init; unbacked rows are zero rows
    Ws, unb = [], []
    for t, w in enumerate(specs):
        W = coracle.init_table(INIT_SEED, w.table.table_id, w.table.hash_size, w.table.dim, 0.1)
        if w.table.elem_bytes == 2:
            W = W.astype(np.float16).astype(np.float32)
        ent = np.asarray(remaps[t].entries)
        u = (ent < 0) & ((-ent.astype(np.int64) - 1) >= remaps[t].slow_rows_allocated)
        W[u] = 0.0
        Ws.append(W)
        unb.append(u)
        assert int(nrows[t]) == int(u.sum())
        lo, hi = int(off[t * B]), int(off[(t + 1) * B])
        assert int(lk[t]) == int(u[idx[lo:hi]].sum()), t
    h = hits.cpu().numpy()
    assert h[0::2].sum() > 0 and h[1::2].sum() > 0
    want, wabs = emb64.forward(B, dims, off, idx, Ws)
    emb64.check(got, want, emb64.RTOL * wabs + 1e-30, "forward")
    for t, w in enumerate(specs):
        rows, g, ga = emb64.row_grads(B, dims, off, idx, got, t)
        backed = ~unb[t][rows]
        wn, mn, wb, mb = emb64.update(Ws[t][rows], np.zeros(rows.size, np.float32), g, ga, opt, lr, 1e-8)
        if w.table.elem_bytes == 2:
            wb = wb + _ulp16(wn)
        gw, gm = op.read_rows(t, rows)
        emb64.check(gw[backed], wn[backed], wb[backed], f"table {t} weights")
        if opt != "sgd":
            emb64.check(gm[backed], mn[backed], mb[backed], f"table {t} momentum")
        assert not gw[~backed].any() and not gm[~backed].any()
        other = np.setdiff1d(np.arange(0, w.table.hash_size, 997, dtype=np.uint32), rows)
        ow, _ = op.read_rows(t, other)
        assert np.array_equal(ow, Ws[t][other])
    op.close()
    return lk


def _rm3_slice():
    """Four RM3-like tables (dim 256, fp16 rows), hash sizes scaled to <= 1e6."""
    specs = wl.rm_specs("rm3", J=12, hash_scale=0.01)
    pick = sorted(range(len(specs)), key=lambda j: -specs[j].gen.mean_pooling * specs[j].gen.coverage)[:4]
    out = [specs[j] for j in sorted(pick)]
    assert all(w.table.elem_bytes == 2 and w.table.dim == 256 for w in out)
    return out


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
def test_rm3_fp16_omit_unaccessed_vs_fp64_oracle(cuda_ctx, coracle, opt, staged):
    lk = _run(cuda_ctx, coracle, _rm3_slice(), 4096, opt, staged, omit=True)
    assert lk.sum() > 0  # unseen rows were looked up


@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
def test_rm3_fp16_fully_backed(cuda_ctx, coracle, opt):
    lk = _run(cuda_ctx, coracle, _rm3_slice(), 2048, opt, False, omit=False)
    assert lk.sum() == 0


@pytest.mark.parametrize("staged", [False, True])
def test_fp32_omit_unaccessed_mixed_dims(cuda_ctx, coracle, staged):
    """fp32 and fp16 tables of several lane classes in one operator, with
    omit_unaccessed remaps."""
    base = wl.rm_specs("rm1", J=6, hash_scale=0.05)
    specs = []
    for j, w in enumerate(base):
        t = w.table
        eb = 2 if j % 2 else 4
        dim = (8, 36, 64, 128, 20, 4)[j]
        specs.append(wl.WorkloadSpec(sp.TableSpec(t.table_id, t.cardinality, t.hash_size, dim, eb), w.gen))
    _run(cuda_ctx, coracle, specs, 2048, "rowwise_adagrad", staged, omit=True)


def test_unbacked_rejected_without_omit(cuda_ctx):
    """A remap whose slow entries reach past slow_rows is rejected unless the
    operator is told those rows are unbacked (rs_emb_table.allow_unbacked)."""
    import ctypes as C

    from paper_2201_10095_b200 import _lib
    from paper_2201_10095_b200.runtime import ptr

    ent = np.array([0, -1, -2, -3], np.int32)
    tabs = (_lib.rs_emb_table * 1)()
    tabs[0] = _lib.rs_emb_table(0, 4, 8, ptr(ent), _lib.RS_MEM_HOST, 1, 1, 2, 0)
    h = C.c_void_p()
    st = _lib.lib().rs_emb_create(cuda_ctx.h, 1, tabs, C.c_uint64(4), C.c_uint64(16), 0, C.c_float(1e-8),
                                  C.byref(h))
    assert st == -1
    tabs[0] = _lib.rs_emb_table(0, 4, 8, ptr(ent), _lib.RS_MEM_HOST, 1, 1, 3, 1)
    st = _lib.lib().rs_emb_create(cuda_ctx.h, 1, tabs, C.c_uint64(4), C.c_uint64(16), 0, C.c_float(1e-8),
                                  C.byref(h))
    assert st == -1  # elem_bytes 3
    tabs[0] = _lib.rs_emb_table(0, 4, 8, ptr(ent), _lib.RS_MEM_HOST, 1, 1, 2, 1)
    _lib.check(_lib.lib().rs_emb_create(cuda_ctx.h, 1, tabs, C.c_uint64(4), C.c_uint64(16), 0,
                                        C.c_float(1e-8), C.byref(h)))
    rows = np.zeros(1, np.uint64)
    _lib.check(_lib.lib().rs_emb_unbacked(h, None, ptr(rows), 0))
    assert rows[0] == 2
    _lib.lib().rs_emb_destroy(h)

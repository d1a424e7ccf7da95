"""GPU parity at BASELINE scale (VERDICT r1 "Next round" 1).

* The tiered EmbeddingBag against the INDEPENDENT fp64 oracle
  (oracle/emb64.py: definition-level sums in float64, FBGEMM exact row-wise
  Adagrad) at 1e-5 relative to each sum's condition, on the full cfg1 batch
  (8 x 1e6 rows, D 64, B 4096, pool 20) and on an RM1 slice at real hash
  sizes (B 16384), both optimizers, zero-copy and pipelined (staged) slow
  tier.  Inputs come from the unmodified reference generator
  (oracle/_ref generate_trace), plans from the GPU profile + remap.
* profile() bit-exact against the unmodified reference profile() on the
  full cfg1 trace (65,536 samples; rates 1.0 and 0.01).
* The partitioned histogram at >= 2^28 ids (multi-chunk buckets) against
  the C oracle; a group whose hottest row overflows the packed rank key
  (table ranges); tables whose hash sizes sum past 2^31 (two counter
  groups) against a sparse numpy count.
"""
import numpy as np
import pytest

import oracle
import paper_2201_10095_b200 as sp
from oracle import emb64
from paper_2201_10095_b200 import workload as wl
from paper_2201_10095_b200.types import PlanEntry, TableSpec, Trace

from conftest import assert_stats_equal

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")]

GEN_SEED = 20260809
INIT_SEED = 1234


def _ref_batch(specs, B, seed=GEN_SEED):
    R = oracle.Ref()
    tr = R.generate_trace([(w.table, (w.gen.zipf_exponent, w.gen.mean_pooling, w.gen.coverage,
                                      w.gen.pooling_law)) for w in specs], B, seed)
    off, idx = oracle.trace_to_csr(tr, [w.table.table_id for w in specs], B)
    trace = Trace([w.table for w in specs], B, tr.rec_sample, tr.rec_table, tr.rec_offset, tr.rec_len,
                  ids=tr.ids)
    R.free_trace(tr)
    return off, idx, trace


def _operator(ctx, specs, trace, frac, B, n, opt):
    stats = sp.profile(trace, 1.0, 7, ctx=ctx)
    remaps = [sp.build_remap(PlanEntry(w.table.table_id, 0, 0, int(frac * st.distinct_rows_accessed)),
                             st, w.table, ctx=ctx) for w, st in zip(specs, stats)]
    op = sp.TieredEmbeddingBag([w.table for w in specs], remaps, B, max(1, n), opt, eps=1e-8, ctx=ctx)
    op.init_weights(INIT_SEED, 0.1)
    return op, remaps


def _check_step(ctx, coracle, specs, B, off, idx, trace, opt, staged, lr):
    import torch

    T = len(specs)
    dims = [w.table.dim for w in specs]
    op, remaps = _operator(ctx, specs, trace, 0.4, B, idx.size, opt)
    d_off = torch.from_numpy(off.astype(np.uint32).view(np.int32)).cuda()
    d_idx = torch.from_numpy(idx.view(np.int32)).cuda()
    if staged:
        slow = sum(int(np.unique(idx[off[t * B]:off[(t + 1) * B]][
            remaps[t].entries[idx[off[t * B]:off[(t + 1) * B]]] < 0]).size) for t in range(T))
        op.enable_uvm_cache(4 * slow + 1024)
        op.prefetch(d_off, d_idx, B)
    hits = torch.zeros(2 * T, dtype=torch.int64, device="cuda")
    y = op.forward(d_off, d_idx, B, hits=hits)
    op.backward(d_off, d_idx, y, B, lr)  # loss 0.5*||pooled||^2: grad = pooled
    if staged:
        op.flush()
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    # both tiers were used
    h = hits.cpu().numpy()
    assert h[0::2].sum() > 0 and h[1::2].sum() > 0
    Ws = [coracle.init_table(INIT_SEED, w.table.table_id, w.table.hash_size, w.table.dim, 0.1)
          for w in specs]
    want, wabs = emb64.forward(B, dims, off, idx, Ws)
    worst = {"forward": emb64.check(got, want, emb64.RTOL * wabs + 1e-30, "forward")}
    for t, w in enumerate(specs):
        rows, g, ga = emb64.row_grads(B, dims, off, idx, got, t)
        wn, mn, wb, mb = emb64.update(Ws[t][rows], np.zeros(rows.size, np.float32), g, ga, opt, lr, 1e-8)
        gw, gm = op.read_rows(t, rows)
        worst[f"w{t}"] = emb64.check(gw, wn, wb, f"table {t} weights")
        if opt != "sgd":
            worst[f"m{t}"] = emb64.check(gm, mn, mb, f"table {t} momentum")
        # untouched rows keep their init
        other = np.setdiff1d(np.arange(0, w.table.hash_size, 9973, dtype=np.uint32), rows)
        ow, _ = op.read_rows(t, other)
        assert np.array_equal(ow, Ws[t][other])
    op.close()
    return worst


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
def test_cfg1_step_vs_fp64_oracle(cuda_ctx, coracle, opt, staged):
    specs = wl.cfg1_specs()
    B = 4096
    off, idx, trace = _ref_batch(specs, B)
    assert idx.size == B * 8 * 20
    _check_step(cuda_ctx, coracle, specs, B, off, idx, trace, opt, staged, lr=0.5)


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("opt", ["sgd", "rowwise_adagrad"])
def test_rm1_slice_step_vs_fp64_oracle(cuda_ctx, coracle, opt, staged):
    """Five RM1-like tables at their real hash sizes (the two largest, up to
    ~1e7 rows, and three heavy-pooling ones), B = 16384."""
    allspecs = wl.rm_specs("rm1")
    by_h = sorted(range(len(allspecs)), key=lambda j: -allspecs[j].table.hash_size)[:2]
    by_pool = sorted(range(len(allspecs)), key=lambda j: -allspecs[j].gen.mean_pooling
                     * allspecs[j].gen.coverage)[:3]
    pick = sorted(set(by_h + by_pool))
    specs = [allspecs[j] for j in pick]
    B = 16384
    off, idx, trace = _ref_batch(specs, B)
    _check_step(cuda_ctx, coracle, specs, B, off, idx, trace, opt, staged, lr=0.5)


@pytest.mark.parametrize("rate", [1.0, 0.01])
def test_profile_full_cfg1_trace_vs_reference(cuda_ctx, rate):
    """the cfg1 8-EMB trace (65,536 samples, 10.5M ids),
    GPU profile() == unmodified reference profile(), every field bit-exact."""
    R = oracle.Ref()
    specs = wl.cfg1_specs()
    tr = R.generate_trace([(w.table, (w.gen.zipf_exponent, w.gen.mean_pooling, w.gen.coverage,
                                      w.gen.pooling_law)) for w in specs], 65536, GEN_SEED)
    want = R.profile(tr, rate, 7)
    got = sp.profile(Trace([w.table for w in specs], 65536, tr.rec_sample, tr.rec_table, tr.rec_offset,
                           tr.rec_len, ids=tr.ids), rate, 7, ctx=cuda_ctx)
    R.free_trace(tr)
    assert_stats_equal(got, want)


def test_profile_partitioned_multichunk_2e28(cuda_ctx, coracle):
    """>= 2^28 ids through the partitioned histogram (buckets of 32768
    counters holding several 1M-address chunks each) == the C oracle."""
    import torch

    specs = wl.cfg1_specs()
    S = (1 << 28) // 160 + 1
    gen = wl.BatchGenerator(specs, S, GEN_SEED + 5, ctx=cuda_ctx)
    off, idx, n = gen.batch(0)
    assert n >= 1 << 28
    tr = wl.kjt_to_trace(specs, off, idx, n, S, 0, ctx=cuda_ctx)
    got = sp.profile(tr, 1.0, 7, ctx=cuda_ctx)
    h = [x.cpu().numpy() for x in (tr.rec_sample, tr.rec_table, tr.rec_offset, tr.rec_len)]
    ids = idx[:n].cpu().numpy().view(np.uint32)
    del idx, off, tr
    torch.cuda.empty_cache()
    want = coracle.profile([w.table for w in specs], S, h[0].view(np.uint64), h[1].view(np.uint32),
                           h[2].view(np.uint64), h[3].view(np.uint32), ids, 1.0, 7)
    assert_stats_equal(got, want)


def _sparse_stats(tables, rec_table, rec_offset, rec_len, ids, num_samples, coracle):
    """profile() at rate 1.0 for traces whose rows are sparse in huge tables:
    np.unique counts, rank (count desc, row asc), cdf = cum/total as doubles
    (core/src/profiler.cpp:125-150), icdf via the C oracle's build_icdf."""
    out = []
    for t in tables:
        sel = rec_table == t.table_id
        lens = rec_len[sel].astype(np.int64)
        st = rec_offset[sel].astype(np.int64)
        pos = np.repeat(st - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
        rows = ids[pos]
        total = int(rows.size)
        pres = int(sel.sum())
        if total:
            u, c = np.unique(rows, return_counts=True)
            order = np.lexsort((u, -c.astype(np.int64)))
            u, c = u[order], c[order].astype(np.uint64)
            cdf = np.cumsum(c).astype(np.float64) / float(total)
            icdf = coracle.build_icdf(c)
        else:
            u, cdf, icdf = np.zeros(0, np.uint32), np.zeros(0), np.zeros(101, np.uint64)
        out.append(dict(table_id=t.table_id, coverage=float(pres) / float(num_samples),
                        avg_pooling=(float(total) / float(pres)) if pres else 0.0,
                        distinct_rows_accessed=int(u.size), total_accesses=total,
                        icdf_steps=icdf, access_cdf=cdf, rows_by_rank=u.astype(np.uint32)))
    return out


def test_profile_hash_sizes_past_2e31_two_groups(cuda_ctx, coracle):
    """Three 8e8-row tables (sum of hash sizes 2.4e9 >= 2^31: two counter
    groups) with Zipf-ish sparse rows == a sparse numpy count."""
    rng = np.random.default_rng(3)
    H = 800_000_000
    tables = [TableSpec(j, H, H, 16, 4) for j in range(3)]
    S = 20000
    rs, rt, ro, rl, ids = [], [], [], [], []
    n = 0
    for s in range(S):
        for j in range(3):
            if rng.random() < 0.7:
                L = int(rng.integers(0, 30))
                rs.append(s), rt.append(j), ro.append(n), rl.append(L)
                head = rng.random(L) < 0.5
                r = np.where(head, rng.integers(0, 1000, L), rng.integers(0, H, L))
                ids.append(r)
                n += L
    ids = np.concatenate(ids).astype(np.uint32)
    rs, rt, ro, rl = (np.array(rs, np.uint64), np.array(rt, np.uint32), np.array(ro, np.uint64),
                      np.array(rl, np.uint32))
    got = sp.profile(Trace(tables, S, rs, rt, ro, rl, ids=ids), 1.0, 7, ctx=cuda_ctx)
    want = _sparse_stats(tables, rt, ro, rl, ids, S, coracle)
    assert_stats_equal(got, want)


def test_profile_rank_key_overflow_splits_tables(cuda_ctx, coracle):
    """4096 tables (12 table bits) and one row counted 1.2M times (21 count
    bits): the packed (table, count) rank key needs 33 bits, so the rank
    runs over table ranges; FeatureStats == the C oracle."""
    J = 4096
    tables = [TableSpec(j, 64, 64, 4, 4) for j in range(J)]
    rng = np.random.default_rng(9)
    rs, rt, ro, rl = [0], [0], [0], [1_200_000]
    ids = [np.zeros(1_200_000, np.int64)]
    n = 1_200_000
    for j in range(1, J):
        L = int(rng.integers(1, 6))
        rs.append(0), rt.append(j), ro.append(n), rl.append(L)
        ids.append(rng.integers(0, 64, L))
        n += L
    ids = np.concatenate(ids).astype(np.uint32)
    tr = Trace(tables, 1, np.array(rs, np.uint64), np.array(rt, np.uint32), np.array(ro, np.uint64),
               np.array(rl, np.uint32), ids=ids)
    got = sp.profile(tr, 1.0, 7, ctx=cuda_ctx)
    want = coracle.profile(tables, 1, tr.rec_sample, tr.rec_table, tr.rec_offset, tr.rec_len, ids, 1.0, 7)
    assert_stats_equal(got, want)

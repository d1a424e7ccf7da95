"""GPU parity: HP1 profiler kernels (K0 hash, K1 histogram, K2 rank/CDF/ICDF)
against the reference goldens and the oracle — bit-exact."""
import numpy as np
import pytest

from conftest import assert_stats_equal, golden_stats, golden_trace, load_golden

import paper_2201_10095_b200 as sp
from paper_2201_10095_b200.types import TableSpec, Trace

pytestmark = pytest.mark.gpu


def test_hash_ids_goldens(cuda_ctx):
    cases = load_golden("hash_value.json")["cases"]
    by_h = {}
    for raw, H, want in cases:
        by_h.setdefault(int(H), []).append((int(raw), int(want)))
    for H, rows in by_h.items():
        if H > 0xFFFFFFFF:
            continue
        raw = np.array([r for r, _ in rows], np.uint64)
        got = sp.hash_ids(raw, H, ctx=cuda_ctx)
        assert list(got) == [w for _, w in rows]


def test_hash_ids_device_large(cuda_ctx, coracle):
    import torch

    rng = np.random.default_rng(1)
    raw = rng.integers(0, 2**63, 1 << 20, dtype=np.int64).astype(np.uint64) * np.uint64(2) + np.uint64(1)
    for H in (1, 7, 1_000_000, 99_999_989, 0x7FFFFFFF):
        got = sp.hash_ids(torch.from_numpy(raw.view(np.int64)).cuda(), H, ctx=cuda_ctx)
        assert np.array_equal(got.cpu().numpy().view(np.uint32), coracle.hash_batch(raw, H))


@pytest.mark.parametrize("name", list(load_golden("profile.json")))
def test_profile_goldens(cuda_ctx, name):
    case = load_golden("profile.json")[name]
    tr = golden_trace(case["trace"], case.get("raw_ids"))
    got = sp.profile(tr, case["rate"], case["seed"], ctx=cuda_ctx)
    assert_stats_equal(got, golden_stats(case["stats"]))


def test_profile_device_trace_and_hash_utilization(cuda_ctx):
    import torch

    case = load_golden("profile.json")["generated_r1.0_s0"]
    tr = golden_trace(case["trace"])
    dev = Trace(tr.tables, tr.num_samples,
                *[torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a.view(np.int32)).cuda()
                  for a in (tr.rec_sample, tr.rec_table, tr.rec_offset, tr.rec_len, tr.ids)])
    got = sp.profile(dev, 1.0, 0, ctx=cuda_ctx)
    assert_stats_equal(got, golden_stats(case["stats"]))
    for st, spec, draw in zip(got, tr.tables, case["distinct_raw"]):
        s, c = sp.hash_utilization(st, spec, draw)
        assert s == (spec.hash_size - st.distinct_rows_accessed) / spec.hash_size
        assert c == (draw - st.distinct_rows_accessed) / spec.hash_size


def test_profile_errors(cuda_ctx):
    case = load_golden("profile.json")["worked_example"]
    tr = golden_trace(case["trace"])
    with pytest.raises(sp.InvalidArgument):
        sp.profile(tr, 0.0, 0, ctx=cuda_ctx)
    with pytest.raises(sp.InvalidArgument):
        sp.profile(tr, 1.5, 0, ctx=cuda_ctx)
    with pytest.raises(sp.InvalidArgument):  # selects zero samples
        sp.profile(tr, 1e-12, 0, ctx=cuda_ctx)
    empty = Trace([], 0, np.zeros(0, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.uint64),
                  np.zeros(0, np.uint32), ids=np.zeros(0, np.uint32))
    with pytest.raises(sp.InvalidArgument):
        sp.profile(empty, 0.5, 0, ctx=cuda_ctx)
    bad = Trace(tr.tables[:1], tr.num_samples, tr.rec_sample, tr.rec_table, tr.rec_offset,
                tr.rec_len, ids=tr.ids)
    with pytest.raises(sp.TableIndexError):  # std::out_of_range, profiler.cpp:103
        sp.profile(bad, 1.0, 0, ctx=cuda_ctx)


def test_build_icdf_goldens(cuda_ctx):
    for case in load_golden("build_icdf.json")["cases"]:
        assert list(sp.build_icdf(case["counts"], ctx=cuda_ctx)) == case["icdf"]
    with pytest.raises(sp.InvalidArgument):
        sp.build_icdf([0, 0, 0], ctx=cuda_ctx)


def _zipf_trace(rng, J, H, S, pool, alpha=1.05):
    """Hashed Zipf trace in the reference layout (records sample-major)."""
    ranks = np.arange(1, 200_001, dtype=np.float64)
    p = ranks ** -alpha
    p /= p.sum()
    tables = [TableSpec(j * 2 + 1, 200_000, H, 64, 4) for j in range(J)]
    R = S * J
    rec_len = np.full(R, pool, np.uint32)
    rec_sample = np.repeat(np.arange(S, dtype=np.uint64), J)
    rec_table = np.tile(np.array([t.table_id for t in tables], np.uint32), S)
    rec_offset = (np.arange(R, dtype=np.uint64) * pool)
    raw = rng.choice(200_000, size=R * pool, p=p).astype(np.uint64)
    return tables, Trace(tables, S, rec_sample, rec_table, rec_offset, rec_len, raw_ids=raw)


def test_profile_large_vs_oracle(cuda_ctx, coracle):
    """cfg1-shaped (8 tables, H=1e6, pooling 20) at 4096 samples, rates 1 and 0.01."""
    rng = np.random.default_rng(7)
    tables, rt = _zipf_trace(rng, 8, 1_000_000, 4096, 20)
    for rate, seed in [(1.0, 0), (0.01, 7), (0.3, 123)]:
        got = sp.profile(rt, rate, seed, ctx=cuda_ctx)  # raw ids hashed on the GPU
        want = coracle.profile(tables, rt.num_samples, rt.rec_sample, rt.rec_table, rt.rec_offset,
                               rt.rec_len, None, rate, seed, raw_ids=rt.raw_ids)
        assert_stats_equal(got, want)


def test_count_distinct_raw(cuda_ctx):
    """GenStats.distinct_raw_ids on the GPU: numpy unique per table, and the
    reference generator's own GenStats when the reference library is present."""
    import oracle

    case = load_golden("profile.json")["raw_trace"]
    tr = golden_trace(case["trace"], case["raw_ids"])
    got = sp.count_distinct_raw(tr, ctx=cuda_ctx)
    for j, t in enumerate(tr.tables):
        mine = tr.rec_table == t.table_id
        vals = np.concatenate([tr.raw_ids[o:o + l] for o, l in zip(tr.rec_offset[mine], tr.rec_len[mine])])
        assert int(got[j]) == np.unique(vals).size
    rng = np.random.default_rng(3)
    tables, rt = _zipf_trace(rng, 3, 50_000, 2000, 7)
    rt.raw_ids[::97] = np.uint64(0xFFFFFFFFFFFFFFFF)  # the hash set's empty sentinel is a valid raw
    got = sp.count_distinct_raw(rt, ctx=cuda_ctx)
    for j, t in enumerate(tables):
        mine = rt.rec_table == t.table_id
        vals = np.concatenate([rt.raw_ids[o:o + l] for o, l in zip(rt.rec_offset[mine], rt.rec_len[mine])])
        assert int(got[j]) == np.unique(vals).size
    if oracle.ref_available():
        R = oracle.Ref()
        S = oracle.Spec
        wl = [(S(0, 5000, 4000, 8, 4), (1.2, 6.0, 0.7, 1)), (S(4, 90000, 30000, 4, 4), (0.8, 3.0, 0.9, 2))]
        ref = R.generate_trace(wl, 4000, 17, gen_stats=True)
        raw = R.generate_trace(wl, 4000, 17, raw=True)
        tr = Trace([TableSpec(**vars(s)) for s in raw.tables], raw.num_samples, raw.rec_sample,
                   raw.rec_table, raw.rec_offset, raw.rec_len, raw_ids=raw.raw_ids)
        assert list(sp.count_distinct_raw(tr, ctx=cuda_ctx)) == list(ref.distinct_raw)


def test_profile_many_tables_and_ragged(cuda_ctx, coracle):
    """Ragged records, empty records, tables never touched, non-contiguous offsets."""
    rng = np.random.default_rng(9)
    J = 37
    tables = [TableSpec(1000 - 7 * j, 10, int(rng.integers(1, 5000)), 4, 4) for j in range(J)]
    S = 3000
    recs = []
    ids = []
    for s in range(S):
        for j in rng.choice(J - 2, size=int(rng.integers(0, 6)), replace=False):
            L = int(rng.integers(0, 40))
            recs.append((s, tables[j].table_id, len(ids), L))
            ids += list(rng.integers(0, tables[j].hash_size, L))
    order = rng.permutation(len(recs))  # offsets stay valid, record order scrambled
    recs = [recs[i] for i in order]
    tr = Trace(tables, S, np.array([r[0] for r in recs], np.uint64),
               np.array([r[1] for r in recs], np.uint32), np.array([r[2] for r in recs], np.uint64),
               np.array([r[3] for r in recs], np.uint32), ids=np.array(ids, np.uint32))
    for rate, seed in [(1.0, 0), (0.5, 3)]:
        got = sp.profile(tr, rate, seed, ctx=cuda_ctx)
        want = coracle.profile(tables, S, tr.rec_sample, tr.rec_table, tr.rec_offset, tr.rec_len,
                               tr.ids, rate, seed)
        assert_stats_equal(got, want)


def test_profile_partitioned_vs_oracle(cuda_ctx, coracle):
    """Calls of >= 2^22 ids with contiguous records take the partitioned
    histogram (P0-P3); ragged/empty records, raw and hashed ids, sampled
    rates.  A scrambled record order (non-contiguous) falls back to the
    atomic kernel.  Bit-exact vs the oracle in every case."""
    import oracle

    rng = np.random.default_rng(31)
    J, S = 6, 120_000
    tables = [TableSpec(j + 3, 100_000, int(h), 16, 4)
              for j, h in enumerate([5_000, 1_000_000, 77_777, 2_000_000, 300, 400_000])]
    lens = rng.integers(0, 15, S * J).astype(np.uint32)  # includes empty records
    lens[::7] = 40
    rec_sample = np.repeat(np.arange(S, dtype=np.uint64), J)
    rec_table = np.tile(np.array([t.table_id for t in tables], np.uint32), S)
    rec_offset = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    N = int(lens.sum())
    assert N >= (1 << 22)
    ranks = np.arange(1, 100_001, dtype=np.float64) ** -1.1
    raw = rng.choice(100_000, size=N, p=ranks / ranks.sum()).astype(np.uint64) * np.uint64(7919)
    tr_raw = Trace(tables, S, rec_sample, rec_table, rec_offset, lens, raw_ids=raw)
    hashed = np.empty(N, np.uint32)
    tab_of = np.repeat(np.tile(np.arange(J), S), lens)
    for j, t in enumerate(tables):
        m = tab_of == j
        hashed[m] = coracle.hash_batch(raw[m], t.hash_size)
    tr_ids = Trace(tables, S, rec_sample, rec_table, rec_offset, lens, ids=hashed)
    for tr, rate, seed in [(tr_ids, 1.0, 0), (tr_raw, 1.0, 5), (tr_ids, 0.3, 9)]:
        got = sp.profile(tr, rate, seed, ctx=cuda_ctx)
        want = coracle.profile(tables, S, rec_sample, rec_table, rec_offset, lens, hashed, rate, seed)
        assert_stats_equal(got, want)
    order = rng.permutation(S * J)
    tr_s = Trace(tables, S, rec_sample[order], rec_table[order], rec_offset[order], lens[order],
                 ids=hashed)
    got = sp.profile(tr_s, 1.0, 0, ctx=cuda_ctx)
    want = coracle.profile(tables, S, rec_sample[order], rec_table[order], rec_offset[order],
                           lens[order], hashed, 1.0, 0)
    assert_stats_equal(got, want)
    del oracle


def test_profile_by_table_shards_equals_whole(cuda_ctx):
    """HP1 across GPUs: each rank profiles the records of its
    tables (sharded.subtrace, device arrays) — the shards' FeatureStats,
    reassembled, equal the whole-trace profile bit for bit.  The ranks run one
    after the other here (one GPU)."""
    import torch

    from paper_2201_10095_b200 import workload as wl
    from paper_2201_10095_b200.sharded import profile_split, subtrace

    specs = wl.rm_specs("rm1", 20260809, J=7, hash_scale=0.01)
    gen = wl.BatchGenerator(specs, 20000, 77)
    off, idx, n = gen.batch(0)
    tr = wl.kjt_to_trace(specs, off, idx, n, 20000, 0, ctx=cuda_ctx)
    # the reference layout: records sorted by (sample, table)
    order = torch.argsort((tr.rec_sample << 32) | (tr.rec_table.long() & 0xFFFFFFFF), stable=True)
    tr = Trace(tr.tables, tr.num_samples, tr.rec_sample[order].contiguous(), tr.rec_table[order].contiguous(),
               tr.rec_offset[order].contiguous(), tr.rec_len[order].contiguous(), ids=tr.ids)
    whole = sp.profile(tr, 0.7, 3, ctx=cuda_ctx)
    for world in (2, 3):
        got = [None] * len(specs)
        for pos in profile_split(tr.tables, world):
            for j, st in zip(pos, sp.profile(subtrace(tr, pos), 0.7, 3, ctx=cuda_ctx)):
                got[j] = st
        assert_stats_equal(got, [vars(s) for s in whole])


def test_profile_partitioned_more_tables_than_shared(cuda_ctx, coracle):
    """The partitioned histogram with more tables than its shared-memory
    table-parameter cache holds (kPSmemTables = 512: the expansion reads base
    and hash size from global memory) and with more than 4096 buckets: 700
    tables, >= 2^22 ids, bit-exact vs the oracle."""
    rng = np.random.default_rng(41)
    J, S = 700, 1500
    tables = [TableSpec(5000 + j, 1000, int(h), 4, 4) for j, h in enumerate(rng.integers(100, 400_000, J))]
    assert sum(t.hash_size for t in tables) > 4096 * 32768
    lens = rng.integers(0, 10, S * J).astype(np.uint32)
    rec_sample = np.repeat(np.arange(S, dtype=np.uint64), J)
    rec_table = np.tile(np.array([t.table_id for t in tables], np.uint32), S)
    rec_offset = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    N = int(lens.sum())
    assert N >= (1 << 22)
    Hs = np.repeat(np.tile(np.array([t.hash_size for t in tables], np.int64), S), lens)
    ids = (rng.random(N) ** 3 * Hs).astype(np.uint32)  # skewed towards low rows
    tr = Trace(tables, S, rec_sample, rec_table, rec_offset, lens, ids=ids)
    got = sp.profile(tr, 1.0, 3, ctx=cuda_ctx)
    want = coracle.profile(tables, S, rec_sample, rec_table, rec_offset, lens, ids, 1.0, 3)
    assert_stats_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("two_pass", [False, True])
def test_profile_partitioned_pool_and_two_pass(cuda_ctx, coracle, monkeypatch, two_pass):
    """The partitioned histogram's two address layouts on the same trace:
    the single-pass chunk pool (few buckets: ids read once, runs appended to
    per-(CTA, bucket) chunks) and, with RS_PROFILE_NO_POOL, the count +
    scatter passes.  Zipf-hot rows, empty records, a 0.4 sample rate;
    bit-exact vs the oracle both ways."""
    if two_pass:
        monkeypatch.setenv("RS_PROFILE_NO_POOL", "1")
    rng = np.random.default_rng(57)
    J, S = 5, 200_000
    tables = [TableSpec(j + 11, 100_000, int(h), 16, 4)
              for j, h in enumerate([3_000_000, 65_536, 1_500_001, 32_767, 900_000])]
    lens = rng.integers(0, 12, S * J).astype(np.uint32)
    lens[::11] = 0
    rec_sample = np.repeat(np.arange(S, dtype=np.uint64), J)
    rec_table = np.tile(np.array([t.table_id for t in tables], np.uint32), S)
    rec_offset = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    N = int(lens.sum())
    assert N >= (1 << 22)
    Hs = np.repeat(np.tile(np.array([t.hash_size for t in tables], np.int64), S), lens)
    ids = (rng.random(N) ** 4 * Hs).astype(np.uint32)
    tr = Trace(tables, S, rec_sample, rec_table, rec_offset, lens, ids=ids)
    for rate, seed in [(1.0, 2), (0.4, 8)]:
        got = sp.profile(tr, rate, seed, ctx=cuda_ctx)
        want = coracle.profile(tables, S, rec_sample, rec_table, rec_offset, lens, ids, rate, seed)
        assert_stats_equal(got, want)


def test_operator_after_big_profile_releases_scratch(cuda_ctx, coracle):
    """A profile whose scratch passes 1 GB (2.5e7 counters), then an operator
    on the same context (its creation releases the context's arena), a
    forward through it, then the same profile again: both profiles
    bit-exact vs the oracle, the forward bit-exact vs the oracle."""
    import torch

    from paper_2201_10095_b200.types import PlanEntry

    rng = np.random.default_rng(71)
    tables = [TableSpec(90 + j, 100, 12_500_000, 16, 4) for j in range(2)]
    S = 30_000
    lens = rng.integers(1, 6, 2 * S).astype(np.uint32)
    rec_sample = np.repeat(np.arange(S, dtype=np.uint64), 2)
    rec_table = np.tile(np.array([90, 91], np.uint32), S)
    rec_offset = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
    N = int(lens.sum())
    ids = (rng.random(N) ** 3 * 12_500_000).astype(np.uint32)
    tr = Trace(tables, S, rec_sample, rec_table, rec_offset, lens, ids=ids)
    want = coracle.profile(tables, S, rec_sample, rec_table, rec_offset, lens, ids, 1.0, 4)
    got = sp.profile(tr, 1.0, 4, ctx=cuda_ctx)
    assert_stats_equal(got, want)
    spec = TableSpec(7, 1000, 5000, 16, 4)
    st = sp.profile(Trace([spec], 1, np.zeros(1, np.uint64), np.full(1, 7, np.uint32), np.zeros(1, np.uint64),
                          np.full(1, 3, np.uint32), ids=np.array([1, 2, 3], np.uint32)), 1.0, 0, ctx=cuda_ctx)[0]
    remap = sp.build_remap(PlanEntry(7, 0, 50, 2), st, spec, ctx=cuda_ctx)
    B = 32
    off = np.arange(0, 2 * B + 1, 2, dtype=np.uint32)
    idx = rng.integers(0, 5000, 2 * B).astype(np.uint32)
    op = sp.TieredEmbeddingBag([spec], [remap], B, idx.size, "sgd", ctx=cuda_ctx)
    op.init_weights(3, 0.5)
    y = op.forward(torch.from_numpy(off.view(np.int32)).cuda(), torch.from_numpy(idx.view(np.int32)).cuda(), B)
    W = [coracle.init_table(3, 7, 5000, 16, 0.5)]
    assert np.array_equal(y.cpu().numpy(), coracle.emb_forward(B, [16], off.astype(np.uint64), idx, W))
    del op
    assert_stats_equal(sp.profile(tr, 1.0, 4, ctx=cuda_ctx), want)

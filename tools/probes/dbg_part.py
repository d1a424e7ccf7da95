import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle
import paper_2201_10095_b200 as sp
from paper_2201_10095_b200.types import TableSpec, Trace
c = oracle.C()
rng = np.random.default_rng(31)
J, S = 6, int(sys.argv[1])
tables = [TableSpec(j + 3, 100_000, int(h), 16, 4) for j, h in enumerate([5_000, 1_000_000, 77_777, 2_000_000, 300, 400_000])]
lens = rng.integers(int(sys.argv[2]), 15, S * J).astype(np.uint32)
lens[::7] = 40
rec_sample = np.repeat(np.arange(S, dtype=np.uint64), J)
rec_table = np.tile(np.array([t.table_id for t in tables], np.uint32), S)
rec_offset = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
N = int(lens.sum())
if len(sys.argv) > 3:
    ranks = np.arange(1, 100_001, dtype=np.float64) ** -1.1
    raw = rng.choice(100_000, size=N, p=ranks / ranks.sum()).astype(np.uint64) * np.uint64(7919)
else:
    raw = rng.integers(0, 1 << 40, N).astype(np.uint64)
hashed = np.empty(N, np.uint32)
tab_of = np.repeat(np.tile(np.arange(J), S), lens)
for j, t in enumerate(tables):
    m = tab_of == j
    hashed[m] = c.hash_batch(raw[m], t.hash_size)
for j, t in enumerate(tables):
    assert hashed[tab_of == j].max() < t.hash_size
if len(sys.argv) > 4:
    tr = Trace(tables, S, rec_sample, rec_table, rec_offset, lens, raw_ids=raw)
else:
    tr = Trace(tables, S, rec_sample, rec_table, rec_offset, lens, ids=hashed)
print("N", N)
try:
    got = sp.profile(tr, 1.0, 0)
    want = c.profile(tables, S, rec_sample, rec_table, rec_offset, lens, hashed, 1.0, 0)
    for g, w in zip(got, want):
        print(g.table_id, g.total_accesses, w["total_accesses"], g.distinct_rows_accessed, w["distinct_rows_accessed"],
              np.array_equal(g.rows_by_rank, w["rows_by_rank"]))
except Exception as e:
    print("ERR", e)

"""K6 on the GPU: the C-ABI exchange (csrc/exchange.cu) driven through
ShardedEmbeddingBag by TWO PROCESSES sharing one GPU (the driver's boxes have
one; CUDA IPC maps each rank's owner block into the other process exactly as
it would across NVLink), with gloo only for the bootstrap.  Every rank's owner
block must equal the single-device oracle forward for its samples (bit-exact:
same fp32 order), and after the backward (gradient = the owner block, written
in place) every rank's tables must equal the oracle's update with the whole
batch's gradients.  Two steps, so both parities of the double buffer run.
NCCL runs at world size 1 in-process; two NCCL ranks on one device are
attempted and skipped when NCCL refuses a duplicate GPU."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = [8, 4, 16, 4, 12, 8, 64]
OWNER = [1, 0, 0, 1, 1, 0, 1]
HS = [300, 50, 1000, 7, 2000, 64, 5000]
SEED, SCALE, LR = 7, 0.5, 0.3


def _batch(B, seed=5):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 7, len(DIMS) * B)
    lens[rng.random(lens.size) < 0.1] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    idx = np.concatenate([np.minimum(rng.zipf(1.3, int(L)) - 1, HS[i // B] - 1)
                          for i, L in enumerate(lens)]).astype(np.uint32)
    return off, idx


def _local_csr(off, idx, tables, B):
    o, parts, base = [0], [], 0
    for t in tables:
        seg = off[t * B:(t + 1) * B + 1]
        parts.append(idx[seg[0]:seg[-1]])
        o.extend((seg[1:] - seg[0] + base).tolist())
        base += int(seg[-1] - seg[0])
    return np.array(o, np.uint32), (np.concatenate(parts) if parts else np.zeros(0, np.uint32))


def _expected(B, steps):
    """Single-device oracle: per step the pooled [B, sum D] and the tables."""
    import oracle
    from paper_2201_10095_b200.types import TableSpec

    c = oracle.C()
    off, idx = _batch(B)
    Ws = [c.init_table(SEED, 40 + j, HS[j], DIMS[j], SCALE) for j in range(len(DIMS))]
    moms = [np.zeros(h, np.float32) for h in HS]
    pooled = []
    for _ in range(steps):
        y = c.emb_forward(B, DIMS, off, idx, Ws)
        pooled.append(y)
        c.emb_backward(B, DIMS, off, idx, y, Ws, moms, 1, LR, 1e-8)
    return off, idx, pooled, Ws, moms


def _run_rank(rank, world, B, transport, steps, q, port=None):
    import torch

    try:
        if world > 1:
            import torch.distributed as dist

            os.environ["MASTER_ADDR"] = "127.0.0.1"
            os.environ["MASTER_PORT"] = str(port)
            os.environ["RS_EXCHANGE_SPIN_LIMIT"] = str(1 << 25)
            dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2201_10095_b200 as sp
        from paper_2201_10095_b200.sharded import ShardedEmbeddingBag
        from paper_2201_10095_b200.types import PlanEntry, ShardingPlan, TableSpec

        owner = OWNER if world > 1 else [0] * len(DIMS)
        plan = ShardingPlan("t", 1, [PlanEntry(40 + j, g, 0, 0) for j, g in enumerate(owner)])
        specs = [TableSpec(40 + j, h, h, d, 4) for j, (h, d) in enumerate(zip(HS, DIMS))]
        mine = [j for j in range(len(DIMS)) if owner[j] == rank]
        remaps = []
        for j in mine:
            H = HS[j]
            rbr = np.random.default_rng(j).permutation(H).astype(np.uint32)
            st = sp.FeatureStats(40 + j, 1.0, 1.0, H, H, np.zeros(101, np.uint64), np.zeros(H), rbr)
            remaps.append(sp.build_remap(PlanEntry(40 + j, rank, 0, H // 2), st, specs[j]))
        off, idx = _batch(B)
        lo, li = _local_csr(off, idx, mine, B)
        d_off = torch.from_numpy(lo.view(np.int32)).cuda()
        d_idx = torch.from_numpy(li.view(np.int32)).cuda()
        sh = ShardedEmbeddingBag(plan, specs, remaps, world, rank, B, max(1, li.size), "rowwise_adagrad",
                                 transport=transport)
        sh.op.init_weights(SEED, SCALE)
        outs = []
        for _ in range(steps):
            y = sh.forward(d_off, d_idx)
            outs.append(y.cpu().numpy().copy())
            sh.backward(d_off, d_idx, LR)  # gradient = the owner block itself
        torch.cuda.synchronize()
        rows = [sh.op.read_rows(t, np.arange(HS[j], dtype=np.uint32)) for t, j in enumerate(mine)]
        sh.close()
        q.put((rank, "ok", outs, mine, rows))
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), None, None))
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _check(results, world, B, steps):
    off, idx, pooled, Ws, moms = _expected(B, steps)
    bl = B // world
    for rank, status, outs, mine, rows in results:
        assert status == "ok", outs
        for k in range(steps):
            want = pooled[k][rank * bl:(rank + 1) * bl]
            assert np.array_equal(outs[k].view(np.uint32), want.view(np.uint32)), (rank, k)
        for (w, m), j in zip(rows, mine):
            assert np.array_equal(w.view(np.uint32), Ws[j].view(np.uint32)), (rank, j)
            assert np.array_equal(m.view(np.uint32), moms[j].view(np.uint32)), (rank, j)


def _spawn(world, B, transport, steps):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, world, B, transport, steps, q, port)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("B", [64, 1000])
def test_peer_exchange_two_ranks_one_gpu(B):
    res = _spawn(2, B, "peer", 2)
    _check(res, 2, B, 2)


def test_nccl_exchange_world1():
    import queue

    q = queue.Queue()
    _run_rank(0, 1, 64, "nccl", 2, q)
    _check([q.get()], 1, 64, 2)


def test_peer_exchange_world1():
    import queue

    q = queue.Queue()
    _run_rank(0, 1, 64, "peer", 2, q)
    _check([q.get()], 1, 64, 2)


def test_nccl_exchange_two_ranks_one_gpu():
    res = _spawn(2, 64, "nccl", 2)
    errs = [r[2] for r in res if r[1] == "error"]
    if errs and any("uplicate" in e or "invalid usage" in e.lower() for e in errs):
        pytest.skip(f"NCCL refuses two ranks on one GPU: {errs[0][:200]}")
    _check(res, 2, 64, 2)

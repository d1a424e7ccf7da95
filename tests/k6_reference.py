"""TEST HELPER — the K6 exchange contract (csrc/exchange.cu) restated with
eager torch.distributed collectives: used by the gloo world-2 test (CPU) and
as the expected layout in the multi-process GPU test.  Rank r owns samples
[r*B/N, (r+1)*B/N); pooled rows arrive in GLOBAL table order; gradients
return as [B, D_local] (this rank's tables in global order)."""
import torch
import torch.distributed as dist

from paper_2201_10095_b200.sharded import column_index, rank_dims


class RefExchange:
    def __init__(self, plan, dims, world, rank, batch, device, group=None):
        self.world, self.rank, self.B, self.bl = world, rank, batch, batch // world
        self.group = group
        self.dims_all = rank_dims(plan, dims, world)
        self.D_local = self.dims_all[rank]
        self.D_total = int(sum(dims))
        self.send_splits = [self.bl * self.D_local] * world
        self.recv_splits = [self.bl * d for d in self.dims_all]
        self._cols = [torch.as_tensor(c, device=device) for c in column_index(plan, dims, world)]
        self.device = device

    def to_owners(self, pooled_local):
        recv = torch.empty(sum(self.recv_splits), dtype=torch.float32, device=self.device)
        src = pooled_local.reshape(-1)[:self.B * self.D_local].contiguous()
        dist.all_to_all_single(recv, src, self.recv_splits, self.send_splits, group=self.group)
        out = torch.empty(self.bl, self.D_total, dtype=torch.float32, device=self.device)
        off = 0
        for s in range(self.world):
            n = self.recv_splits[s]
            if n:
                out[:, self._cols[s]] = recv[off:off + n].view(self.bl, self.dims_all[s])
            off += n
        return out

    def to_tables(self, grad_owned):
        parts = [grad_owned[:, self._cols[s]].reshape(-1) for s in range(self.world) if self.dims_all[s]]
        send = torch.cat(parts)
        out = torch.empty(self.B * self.D_local, dtype=torch.float32, device=self.device)
        dist.all_to_all_single(out, send.contiguous(), self.send_splits, self.recv_splits, group=self.group)
        return out.view(self.B, self.D_local)

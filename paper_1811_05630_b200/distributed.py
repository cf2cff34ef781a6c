"""Multi-GPU slice sharding over torch.distributed.

One process per GPU.  Slice j lives on rank j // (S / world): the top
log2(world) slice-index bits are the rank bits, every slice keeps the
reference layout, so per-slice QCB1 streams are bit-identical for any world
size.  Per gate:

  * X1 exchange -- a butterfly / swap whose partner mask touches rank bits
    pairs every local slice with a slice on ONE partner rank
    (rank ^ (mask >> log2 ns)); both ranks ship their compressed slices
    (QCB1 bytes, not dense amplitudes) with one batched isend/irecv, and each
    side re-encodes only its own slices;
  * X2 norms -- every rank's per-slice sq_norm table is all-gathered before
    the next gate so every rank computes the identical scale 1/sqrt(G)
    (deterministic tree sum over all slices).

The backend is whatever the process group uses: NCCL over NVLink/NVSwitch
on the GPU box (tensors staged on the device), gloo in the CPU tests, where
the oracle engine stands in for the device engine behind the same hooks.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def partner_mask(action, s: int) -> int:
    """Slice-index XOR mask of the partner slice."""
    if action.kind == 1 and action.target >= s:
        return 1 << (action.target - s)
    if action.kind == 2:
        return (1 << (action.a - s) if action.a >= s else 0) | (1 << (action.b - s) if action.b >= s else 0)
    return 0


class ShardedEngine:
    def __init__(self, config=None, engine=None, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if engine is None:
            from .engine import Engine
            config.rank, config.world = self.rank, self.world
            engine = Engine(config)
        self.eng = engine
        self.n, self.s = engine.n, engine.s
        self.S = 1 << (self.n - self.s)
        if self.S % self.world:
            raise ValueError("slice count must be divisible by the world size")
        self.ns = self.S // self.world
        self.s0 = self.rank * self.ns
        self.log2ns = self.ns.bit_length() - 1
        backend = dist.get_backend(group)
        self.dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        self.exchanged_bytes = 0

    # -------------------------------------------------------------- norms
    def _sync_norms(self):
        local = torch.from_numpy(np.ascontiguousarray(self.eng.slice_norms())).to(self.dev)
        out = [torch.empty_like(local) for _ in range(self.world)]
        dist.all_gather(out, local, group=self.group)
        self.eng.set_global_norms(torch.cat(out).cpu().numpy())

    def load_basis(self, x: int):
        self.eng.load_basis(x)
        self._sync_norms()

    def load_amplitudes(self, amps):
        self.eng.load_amplitudes(amps)
        self._sync_norms()

    # ----------------------------------------------------------- exchange
    def _exchange(self, action):
        hm = partner_mask(action, self.s)
        rbits = hm >> self.log2ns
        if rbits == 0:
            return
        peer = self.rank ^ rbits
        # the peer's partners are exactly my slices (XOR with a rank bit maps
        # its range onto mine)
        mine = [self.s0 + k for k in range(self.ns)]
        if self.dev.type == "cuda" and hasattr(self.eng, "export_slices_device"):
            self._exchange_device(mine, peer)
            return
        if hasattr(self.eng, "export_slices"):
            buf, offs = self.eng.export_slices(mine)
            blob = np.asarray(buf, dtype=np.uint8)
            lens_l = [offs[k + 1] - offs[k] for k in range(self.ns)]
        else:  # oracle engine (CPU tests)
            blobs = [self.eng.export_slice(j) for j in mine]
            blob = np.frombuffer(b"".join(blobs), dtype=np.uint8)
            lens_l = [len(b) for b in blobs]
        lens = torch.tensor(lens_l, dtype=torch.int64, device=self.dev)
        rlens = torch.empty_like(lens)
        ops = [dist.P2POp(dist.isend, lens, peer, self.group), dist.P2POp(dist.irecv, rlens, peer, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        payload = torch.from_numpy(blob.copy()).to(self.dev)
        rbuf = torch.empty(int(rlens.sum().item()), dtype=torch.uint8, device=self.dev)
        ops = [dist.P2POp(dist.isend, payload, peer, self.group), dist.P2POp(dist.irecv, rbuf, peer, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        data = rbuf.cpu().numpy().tobytes()
        self.exchanged_bytes += payload.numel()
        p0 = peer * self.ns
        off = 0
        for k, ln in enumerate(rlens.cpu().tolist()):
            self.eng.import_partner(p0 + k, data[off:off + ln])
            off += ln

    def _exchange_device(self, mine, peer):
        """X1 without host staging: the engine gathers my slices' blocks into
        a device tensor, NCCL ships it to the peer, the peer's engine decodes
        straight from the received device buffer."""
        total, offs = self.eng.export_slices_device(mine)
        buf = torch.empty(max(1, total), dtype=torch.uint8, device=self.dev)
        self.eng.export_slices_device(mine, buf.data_ptr(), buf.numel())
        meta = torch.tensor(offs, dtype=torch.int64, device=self.dev)
        rmeta = torch.empty_like(meta)
        ops = [dist.P2POp(dist.isend, meta, peer, self.group), dist.P2POp(dist.irecv, rmeta, peer, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        roffs = rmeta.cpu().tolist()
        rbuf = torch.empty(max(1, roffs[-1]), dtype=torch.uint8, device=self.dev)
        ops = [dist.P2POp(dist.isend, buf, peer, self.group), dist.P2POp(dist.irecv, rbuf, peer, self.group)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        torch.cuda.current_stream(self.dev).synchronize()  # the engine's stream reads rbuf next
        self.exchanged_bytes += total
        self.eng.import_partners_device([peer * self.ns + k for k in range(self.ns)], rbuf.data_ptr(), roffs)
        self._keep = rbuf  # alive until the gate has run

    def run(self, actions=()):
        for a in actions:
            self._exchange(a)
            self.eng.run([a])
            self._sync_norms()
        return self.metrics()

    # ------------------------------------------------------------ metrics
    def metrics(self):
        m = self.eng.run([]) if not hasattr(self.eng, "metrics") else self.eng.metrics()
        peak = m.peak_compressed_bytes
        if hasattr(self.eng, "gate_metrics"):
            # global peak = max over passes of the SUM over ranks (every rank
            # runs the same passes since its load)
            per = torch.tensor([float(r["bytes"]) for r in self.eng.gate_metrics()], dtype=torch.float64,
                               device=self.dev)
            dist.all_reduce(per, op=dist.ReduceOp.SUM, group=self.group)
            peak = int(per.max().item()) if per.numel() else 0
        t = torch.tensor([m.min_compression_ratio, m.mean_compression_ratio * m.compress_calls, m.compress_calls,
                          m.current_compressed_bytes, 0.0, m.wall_seconds],
                         dtype=torch.float64, device=self.dev)
        mn = t[0:1].clone()
        dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=self.group)
        sm = t[1:5].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM, group=self.group)
        mx = t[5:6].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=self.group)
        m.min_compression_ratio = float(mn.item())
        calls = float(sm[1].item())
        m.mean_compression_ratio = float(sm[0].item()) / calls if calls else 0.0
        m.compress_calls = int(calls)
        m.current_compressed_bytes = int(sm[2].item())
        m.peak_compressed_bytes = peak if hasattr(self.eng, "gate_metrics") else int(m.peak_compressed_bytes)
        m.wall_seconds = float(mx.item())
        return m

    def slice_norms(self):
        return self.eng.slice_norms()

    def export_local_blocks(self) -> bytes:
        return self.eng.export_blocks()[0]

    def gather_blocks(self) -> bytes:
        """All ranks' blocks in global plane order (testing / checkpoints)."""
        objs = [None] * self.world
        dist.all_gather_object(objs, self.export_local_blocks(), group=self.group)
        return b"".join(objs)

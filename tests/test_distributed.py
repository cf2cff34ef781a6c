"""Multi-rank slice sharding over torch.distributed (gloo, world size 2 and
4, CPU).  The oracle engine stands in for the device engine behind the same
hooks; the sharded run must be byte-identical to the single-process run
("regardless of worker count")."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    # name: (n, s, circuit)
    "qft9": (9, 4, "qft"),
    "grover8": (8, 3, "grover"),
    "mixed": (8, 3, "mixed"),
}


def _actions(which, n):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1811_05630_b200.circuit as c
    if which == "qft":
        return c.lower(c.build_qft(n))
    if which == "grover":
        return c.lower(c.build_grover(n, 0b10110101 & ((1 << n) - 1), 2))
    G = c.Gate
    gates = [G.h(q) for q in range(n)] + [G.swap(0, 7), G.swap(6, 7), G.cnot(7, 1), G.cnot(0, 6), G.y(7),
                                          G.cphase(0.4, 6, 7), G.mcz([1, 6, 7]), G.swap(2, 5)]
    return [c.to_action_c(c.gate_action(g)) for g in gates]


def _worker(rank, world, port, name, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import CodecConfig, EngineConfig, Oracle
    from paper_1811_05630_b200.distributed import ShardedEngine
    n, s, which = CASES[name]
    acts = _actions(which, n)
    eng = Oracle().engine(EngineConfig.make(n, s, CodecConfig.make(1, 1e-5, 16, 0), rank=rank, world=world))
    se = ShardedEngine(engine=eng)
    se.load_basis(0 if which != "qft" else 77)
    m = se.run(acts)
    blocks = se.gather_blocks()
    if rank == 0:
        out.put((blocks, m.min_compression_ratio, m.compress_calls, se.exchanged_bytes))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", list(CASES))
def test_sharded_equals_single(oracle, name, world):
    from oracle.oracle import CodecConfig, EngineConfig
    n, s, which = CASES[name]
    acts = _actions(which, n)
    single = oracle.engine(EngineConfig.make(n, s, CodecConfig.make(1, 1e-5, 16, 0)))
    single.load_basis(0 if which != "qft" else 77)
    ms = single.run(acts)
    want = single.export_blocks()[0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _port(), name, q), nprocs=world, join=True, start_method="spawn")
    blocks, mn, calls, xbytes = q.get(timeout=60)
    assert blocks == want
    assert mn == ms.min_compression_ratio
    assert calls == ms.compress_calls
    assert xbytes > 0  # gates on rank bits really exchanged compressed slices

"""Host-side logic of the multi-GPU path on CPU (no GPU needed): world_size-2 `gloo`
process groups check that the block-cyclic layout (include/stepfact.h, sf_local_cols;
the binding's scatter/gather) partitions the columns exactly as DESIGN.md §8 states, and
that every rank derives the same panel ownership from (n, s, G) alone — which is what
lets each rank enqueue the same broadcast sequence without negotiating it."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_1812_02056_b200 as sf  # noqa: E402
from paper_1812_02056_b200 import build as sfbuild  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for n, s in cases:
            nloc = sf.local_cols(n, s, world, rank)
            cols = sf.global_columns(n, s, world, rank)
            assert nloc == len(cols)
            # panels owned: p = rank, rank + G, ... ; local column slot*s + k is global p*s + k
            for j, g in enumerate(cols):
                p = g // s
                assert p % world == rank and (p // world) * s + g % s == j
            allc = [None] * world
            dist.all_gather_object(allc, cols)
            flat = sorted(c for cs in allc for c in cs)
            assert flat == list(range(n)), "columns must be partitioned exactly"
            # scatter -> all_gather -> gather reproduces the matrix
            rng = np.random.default_rng(n * 7 + s)
            B = torch.from_numpy(rng.standard_normal((n, n)))      # column-major buffer, same on all ranks
            X = sf.scatter_cyclic(B, n, s, world, rank)
            sizes = [sf.local_cols(n, s, world, r) for r in range(world)]
            pieces = [torch.zeros(sz, n, dtype=B.dtype) for sz in sizes]
            Xp = torch.zeros(max(sizes), n, dtype=B.dtype); Xp[:nloc] = X
            gathered = [torch.zeros(max(sizes), n, dtype=B.dtype) for _ in range(world)]
            dist.all_gather(gathered, Xp)
            for r in range(world):
                pieces[r] = gathered[r][:sizes[r]]
            Y = torch.zeros_like(B)
            sf.gather_cyclic(pieces, n, s, world, Y)
            assert torch.equal(Y, B)
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_block_cyclic_layout_gloo_world2():
    sfbuild.build()
    cases = [(1, 1), (10, 3), (64, 16), (130, 32), (300, 64), (1000, 168), (96, 96)]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


@pytest.mark.parametrize("n,s,G", [(65536, 512, 8), (65536, 512, 3), (8192, 128, 2), (16384, 168, 4)])
def test_local_cols_formula(n, s, G):
    P = -(-n // s)
    widths = [min(s, n - p * s) for p in range(P)]
    for r in range(G):
        assert sf.local_cols(n, s, G, r) == sum(widths[r::G])
    assert sum(sf.local_cols(n, s, G, r) for r in range(G)) == n
    assert sf.local_cols(n, s, G, G) == 0 and sf.local_cols(n, s, G, -1) == 0

"""Multi-process (world size 2, gloo, CPU) tests of the multi-GPU host logic.

* batch sharding: rows split without gaps/overlap, every rank's rows
  transformed independently, gathered result == oracle on the whole batch;
* sharded four-step orchestration (dist.fft_dist): scatter -> phase 0 ->
  all_to_all_single over gloo -> phase 1 -> gather, with the two GPU phases
  replaced by a numpy model of the same data layouts (the GPU kernels behind
  the phases are checked in tests/test_gpu_dist.py).  The model uses numpy's
  FFT as a stand-in inside this CPU-only test; the result is checked against
  the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_07264_b200 import dist as sdist


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def model_phase(m, world, rank):
    l1 = m // 2
    n1, n2 = 1 << l1, 1 << (m - l1)

    def phase(ph, xr, xi):
        x = (np.asarray(xr, dtype=np.float64) + 1j * np.asarray(xi, dtype=np.float64))
        if ph == 0:
            xl = x.reshape(n1, n2 // world)                     # [n1][n2 local]
            y = np.fft.fft(xl, axis=0)                          # [k1][n2 local]
            send = y.reshape(world, n1 // world, n2 // world).transpose(0, 2, 1)  # [h][n2l][k1l]
            out = send.reshape(-1)
        else:
            z = x.reshape(n2, n1 // world)                      # [n2][k1 local]
            k1 = rank * (n1 // world) + np.arange(n1 // world)
            nn2 = np.arange(n2)
            tw = np.exp(-2j * np.pi * np.outer(nn2, k1) / (n1 * n2))
            out = np.fft.fft(z * tw, axis=0).reshape(-1)        # [k2][k1 local]
        return torch.from_numpy(out.real.copy()), torch.from_numpy(out.imag.copy())
    return phase


def worker(rank, world, port, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)
        xr = rng.standard_normal(1 << m)
        xi = rng.standard_normal(1 << m)
        l1 = m // 2
        lr = torch.from_numpy(np.ascontiguousarray(sdist.scatter_input(xr, world, rank, l1)))
        li = torch.from_numpy(np.ascontiguousarray(sdist.scatter_input(xi, world, rank, l1)))
        yr, yi = sdist.fft_dist(lr, li, m=m, phase_fn=model_phase(m, world, rank))
        outs = [None] * world
        dist.all_gather_object(outs, (yr.numpy(), yi.numpy()))
        if rank == 0:
            gr = sdist.gather_output([o[0] for o in outs], l1)
            gi = sdist.gather_output([o[1] for o in outs], l1)
            q.put((gr, gi))
        # batch sharding
        b = 37
        start, end = sdist.shard_rows(b, world, rank)
        rows = [None] * world
        dist.all_gather_object(rows, (start, end))
        if rank == 0:
            q.put(rows)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [12, 14])
def test_four_step_orchestration_world2(m):
    from oracle import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    gr, gi = q.get(timeout=120)
    rows = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(42)
    xr = rng.standard_normal(1 << m)
    xi = rng.standard_normal(1 << m)
    wr, wi = oracle.fft_split_c(xr, xi)
    scale = 1 + np.abs(wr).max()
    assert np.max(np.abs(gr - wr)) <= 1e-9 * scale and np.max(np.abs(gi - wi)) <= 1e-9 * scale
    assert rows == [(0, 19), (19, 37)]


def test_shard_rows_cover_the_batch():
    for b in (0, 1, 7, 1 << 20):
        for w in (1, 2, 3, 8):
            spans = [sdist.shard_rows(b, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == b
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1
    with pytest.raises(ValueError):
        sdist.shard_rows(8, 2, 2)


def test_layout_helpers_round_trip():
    m, world = 10, 4
    l1 = m // 2
    x = np.arange(1 << m)
    blocks = [sdist.scatter_input(x, world, r, l1) for r in range(world)]
    # rank r owns n2 in [r*N2/G, (r+1)*N2/G) for every n1
    n2 = 1 << (m - l1)
    for r, blk in enumerate(blocks):
        assert blk.shape == (1 << l1, n2 // world)
        assert np.all((blk % n2) // (n2 // world) == r)
    # gather: rank h holds [k2][k1 local]
    outs = [np.arange(h * 8, h * 8 + 8)[None, :] + 32 * np.arange(32)[:, None] for h in range(world)]
    g = sdist.gather_output(outs, l1)
    assert np.array_equal(g, np.arange(1 << m))

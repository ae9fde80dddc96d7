"""Row-sharded matching (rowshard.match_rows_sharded) over gloo on CPU with an
exact float64 numpy nearest search standing in for the GPU one: world 1, 2, 3
must all reproduce the oracle's match list bit-exactly, including duplicate
rows split across ranks (global first-argmin ties)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lpsift_oracle as O
from paper_2405_08578_b200.rowshard import match_rows_sharded


def cpu_nearest(X, Y):
    idx = np.empty(X.shape[0], np.int64)
    dd = np.empty(X.shape[0])
    Yn = Y.double().numpy()
    for i0, D in O.distances(X.double().numpy(), Yn):
        j = np.argmin(D, axis=1)
        idx[i0:i0 + D.shape[0]] = j
        dd[i0:i0 + D.shape[0]] = D[np.arange(D.shape[0]), j]
    return torch.from_numpy(idx.astype(np.int32)), torch.from_numpy(dd)


def data():
    rng = np.random.default_rng(4)
    A = rng.random((90, 128)).astype(np.float32)
    A /= np.linalg.norm(A, axis=1, keepdims=True)
    B = (A[rng.permutation(90)[:70]] + rng.normal(0, 0.01, (70, 128))).astype(np.float32)
    A[50] = A[3]  # identical rows on different ranks
    A[80] = A[3]
    B[10] = B[11]
    return torch.from_numpy(A), torch.from_numpy(B)


def shards(n, world):
    b = np.linspace(0, n, world + 1).astype(int)
    return [(int(b[r]), int(b[r + 1])) for r in range(world)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B = data()
        lo, hi = shards(A.shape[0], world)[rank]
        r1, r2, dl = match_rows_sharded(A[lo:hi], lo, B, 0.35, nearest_fn=cpu_nearest)
        q.put((rank, r1.numpy(), r2.numpy(), dl.numpy()))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_matches():
    A, B = data()
    return O.match(A.double().numpy(), B.double().numpy(), 0.35)


def test_single_process_equals_oracle():
    A, B = data()
    r1, r2, dl = match_rows_sharded(A, 0, B, 0.35, nearest_fn=cpu_nearest)
    w1, w2, wd = oracle_matches()
    assert np.array_equal(r1.numpy(), w1) and np.array_equal(r2.numpy(), w2) and np.array_equal(dl.numpy(), wd)
    assert len(w1) > 20


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_equal_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    w1, w2, wd = oracle_matches()
    for _ in procs:
        rank, r1, r2, dl = q.get(timeout=10)
        assert np.array_equal(r1, w1) and np.array_equal(r2, w2) and np.array_equal(dl, wd), rank

"""The row-sharded (multi-GPU) path on CPU with torch.distributed gloo,
world size 2: the partition and NCCL-id exchange the bench
uses (paper_1509_00296_b200.sharding), and the contraction structure of the
library's sharded FRSVT — local sketch / A Z / composition, all-reduced
Grams and A^T Q, replicated small factors — emulated in fp64 numpy per rank
and gathered, against the single-process oracle (tolerance 1e-10)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1509_00296_b200.sharding import exchange_unique_id, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _orth_sharded(Yk):
    """CholeskyQR2 of a row-sharded Y: all-reduced fp64 Gram, replicated factor."""
    for _ in range(2):
        G = _allreduce(Yk.T @ Yk)
        R = np.linalg.cholesky(G).T
        Yk = np.linalg.solve(R.T, Yk.T).T
    return Yk


def _frsvt_sharded(Ak, Omega, q, tau):
    """Alg. 1 (no RP) with the library's sharding: returns this rank's rows of X."""
    Qk = _orth_sharded(Ak @ Omega)                 # local sketch, reduced Gram
    for _ in range(q):
        Z = _allreduce(Ak.T @ Qk)                  # A^T Q: reduction over rows
        Zq = np.linalg.qr(Z)[0]                    # replicated (Z is replicated)
        Qk = _orth_sharded(Ak @ Zq)                # local A Z
    Bt = _allreduce(Ak.T @ Qk)                     # B^T = A^T Q
    G = Bt.T @ Bt                                  # replicated l x l Gram B B^T
    lam, U = np.linalg.eigh(G)
    sig = np.sqrt(np.maximum(lam, 0.0))
    f = np.where(sig > tau, (sig - tau) / np.where(sig > 0, sig, 1.0), 0.0)
    return (Qk @ (U * f)) @ (U.T @ Bt.T)           # local composition


def _worker(rank, ws, port, A, Omega, q, tau, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        uid = exchange_unique_id(dist, rank, lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        row0, mloc = shard(A.shape[0], ws, rank)
        Xk = _frsvt_sharded(A[row0:row0 + mloc], Omega, q, tau)
        # the replicated small results agree bit for bit across ranks
        chk = torch.tensor([float(np.sum(Xk)), float(mloc)], dtype=torch.float64)
        parts = [torch.zeros(2, dtype=torch.float64) for _ in range(ws)]
        dist.all_gather(parts, chk)
        out[rank] = (row0, Xk)
        if rank == 0:
            assert sum(int(p[1]) for p in parts) == A.shape[0]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,ws", [(10, 3), (7, 2), (1, 1), (65536, 8), (76800, 8)])
def test_shard_partition(m, ws):
    rows = []
    for r in range(ws):
        row0, ml = shard(m, ws, r)
        rows.extend(range(row0, row0 + ml))
        assert abs(ml - m // ws) <= 1
    assert rows == list(range(m))
    with pytest.raises(ValueError):
        shard(m, ws, ws)


def test_sharded_frsvt_matches_oracle():
    import oracle

    rng = np.random.default_rng(3)
    m, n, l, q, ws = 157, 64, 12, 1, 2
    A = (rng.standard_normal((m, 6)) * np.logspace(1, 0, 6)) @ rng.standard_normal((6, n)) \
        + 1e-3 * rng.standard_normal((m, n))
    Omega = rng.standard_normal((n, l))
    tau = 2.0
    ref = oracle.frsvt(A, Omega, l, q, tau=tau, rp=False)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(ws, _free_port(), A, Omega, q, tau, out), nprocs=ws, join=True)
        X = np.zeros_like(A)
        for r in range(ws):
            row0, Xk = out[r]
            X[row0:row0 + Xk.shape[0]] = Xk
    assert np.linalg.norm(X - ref.X) <= 1e-10 * np.linalg.norm(ref.X)

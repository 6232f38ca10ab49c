"""Host-side logic of the row-sharded (multi-GPU) path, SURVEY.md §8(e).

Rank k of N holds rows [row0, row0 + m_local) of every m-row operand (A or
D, E, the ALM operand, Y, Q, Q~). Products whose reduction runs over rows
(Grams Y^T Y, A^T Q, the residual) are all-reduced inside libfrsvt with NCCL
on the handle's stream; everything derived from reduced data (Omega,
orth(Z), the Cholesky factors, the small SVD, the shrink) is computed
redundantly and bit-identically on every rank. This module holds only the
partition and the NCCL-id exchange; the library does the rest.
"""


def shard(m, ws, rank):
    """(row0, m_local) of `rank`: contiguous, balanced to within one row."""
    if ws < 1 or not 0 <= rank < ws:
        raise ValueError("bad rank %d of %d" % (rank, ws))
    base, rem = divmod(int(m), ws)
    m_loc = base + (1 if rank < rem else 0)
    row0 = rank * base + min(rank, rem)
    return row0, m_loc


def exchange_unique_id(dist, rank, make_id):
    """Rank 0 creates the 128-byte NCCL unique id with `make_id()` and every
    rank receives it through the torch.distributed process group."""
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("NCCL unique id must be 128 bytes")
    return bytes(uid)

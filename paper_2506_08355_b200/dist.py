"""One process per GPU: NCCL bootstrap over torch.distributed and the rank's slice of a problem.

torch.distributed is plumbing only (it carries the 128-byte ncclUniqueId from rank 0 and the
final max-over-ranks timing); every data-path collective of the partitioned solve (Gram
allreduces, halo exchange, X allgather) runs inside libbosp_b200.so on its own NCCL
communicator (csrc/comm.cpp NcclComm).
"""
from __future__ import annotations

import numpy as np

from . import bosp


def broadcast_uid(make_uid=bosp.comm_nccl_unique_id) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    import torch.distributed as dist
    obj = [make_uid() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def attach(op, uid: bytes, nranks: int, rank: int):
    """Attach the NCCL communicator and this rank's row window (bosp.row_slice rule of the global
    operator `op`) to the calling thread; returns (row0, n_local)."""
    row0, nl, _, _ = bosp.row_slice(op, nranks, rank)
    n = op.n if not isinstance(op, np.ndarray) else op.shape[0]
    bosp.comm_init_nccl(uid, nranks, rank, n, row0)
    return row0, nl


def local_nullspace(x0, y0, row0, nl):
    """This rank's rows of a global (X0, Y0)."""
    return bosp.GeneralizedNullspace(np.asfortranarray(x0[row0:row0 + nl]), np.asfortranarray(y0[row0:row0 + nl]))


def halo_columns(rowptr, colidx, row0, nl):
    """Global columns outside [row0, row0 + nl) that this rank's CSR rows touch, sorted and
    unique: the rows it receives per apply (the plan CsrRowsOp builds, operators.cpp)."""
    a, b = int(rowptr[row0]), int(rowptr[row0 + nl])
    c = np.unique(np.asarray(colidx[a:b]))
    return c[(c < row0) | (c >= row0 + nl)]

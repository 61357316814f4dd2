"""Host logic of the row-partitioned path, two ranks over gloo on CPU (world_size 2).

Covers what runs on the host when bench.py / a user launches one process per GPU: the NCCL
unique-id broadcast, the row-slice rule (bosp.row_slice == multi.cpp row_slice), the halo plan
of a CSR slice (the columns CsrRowsOp receives; one z-plane per neighbour for the 7-point
operator), and that local partial Grams allreduce to the global Gram -- checked with numpy on
the same seeded data.  The device side of the same path is tests/test_gpu_multi.py.
"""
import os
import socket

import numpy as np
import pytest

from paper_2506_08355_b200 import bosp, dist as D
from paper_2506_08355_b200 import problems as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problems():
    kop, mop = P._grid3_ops(6)
    return {
        "t101": (P.t_matrix(101, 0.0), P.t_matrix(101, 0.0)),
        "grid3": (kop, mop),
        "grid2": (P.Stencil(9, 7, 1, "neumann", 1.0), P.Stencil(9, 7, 1, "dirichlet", 1.0, "harmonic", -3.0, 0.5)),
    }


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = D.broadcast_uid(make_uid=lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        for name, (k, m) in _problems().items():
            for op in (k, m):
                csr = op.to_csr() if isinstance(op, P.Stencil) else op
                n = csr.n
                row0, nl, s0, cnt = bosp.row_slice(op, world, rank)
                slices = [None] * world
                dist.all_gather_object(slices, (row0, nl))
                assert slices[0][0] == 0 and sum(s[1] for s in slices) == n
                assert all(slices[i][0] + slices[i][1] == slices[i + 1][0] for i in range(world - 1))
                if isinstance(op, P.Stencil):
                    plane = op.nx * op.ny if op.nz > 1 else op.nx
                    assert row0 == s0 * plane and nl == cnt * plane
                # halo plan: one boundary plane per neighbour for the stencils
                halo = D.halo_columns(csr.rowptr, csr.colidx, row0, nl)
                if isinstance(op, P.Stencil):
                    plane = op.nx * op.ny if op.nz > 1 else op.nx
                    assert halo.size == plane * (world - 1)
                # partitioned apply: owned rows of x plus received halo rows only
                rng = np.random.default_rng(7)
                x = rng.uniform(-1, 1, (n, 3))
                x_local = x[row0:row0 + nl]
                parts = [None] * world
                dist.all_gather_object(parts, (row0, x_local))
                x_seen = np.zeros_like(x)
                x_seen[row0:row0 + nl] = x_local
                for r0, xl in parts:
                    idx = halo[(halo >= r0) & (halo < r0 + xl.shape[0])]
                    x_seen[idx] = xl[idx - r0]
                a = csr.scipy()
                y_local = a[row0:row0 + nl] @ x_seen
                ys = [None] * world
                dist.all_gather_object(ys, y_local)
                assert np.allclose(np.vstack(ys), a @ x, rtol=0, atol=1e-12)
                # Gram allreduce: local partial X^T Y summed over ranks == global X^T Y
                y = rng.uniform(-1, 1, (n, 4))
                g = torch.from_numpy(x_local.T @ y[row0:row0 + nl])
                dist.all_reduce(g)
                assert np.allclose(g.numpy(), x.T @ y, rtol=1e-13, atol=1e-13)
        out.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        out.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_partition_host_logic_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}


@pytest.mark.parametrize("nranks", [1, 2, 3, 5, 8])
def test_row_slice_tiles_rows(nranks):
    for op in (P.t_matrix(37, 0.0), P.Stencil(4, 5, 6, "neumann", 1.0), P.Stencil(5, 11, 1, "neumann", 1.0)):
        n = op.n
        spans = [bosp.row_slice(op, nranks, r) for r in range(nranks)]
        assert spans[0][0] == 0 and sum(s[1] for s in spans) == n
        assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(nranks - 1))

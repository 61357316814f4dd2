"""B200-native BOSP core (arxiv 2506.08355): fp64 SpMM / DMMA tall-skinny GEMMs / MGS-Biorth
kernels for sm_100a behind the reference's solver + matvec-callback API.

    from paper_2506_08355_b200 import bosp
    K = bosp.LinearOperator.from_csr(rowptr, colidx, vals)
    res = bosp.solve(K, M, bosp.InnerProduct(), bosp.BospConfig(nev=20, nb=40), ns)
"""
__all__ = ["bosp", "problems"]

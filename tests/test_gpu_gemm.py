"""FP64 matmul on the GPU: the bit-exact seam against reference fixtures, the
DMMA DGEMM against host float64 (rel-L2 <= 1e-12, the stated fp64 bar)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["m1", "m2", "m3"])
def test_matmul_seam_bitwise(name):
    import torch

    from paper_2506_02486_b200 import kernels
    g = np.load(os.path.join(GOLDEN, "kernels_golden.npz"))
    a = torch.from_numpy(g[f"{name}_a"]).cuda()
    b = torch.from_numpy(g[f"{name}_b"]).cuda()
    c = torch.empty(a.shape[0], b.shape[1], dtype=torch.float64, device="cuda")
    kernels.matmul_f64(a, b, c)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy().view(np.uint64), g[f"{name}_c"].view(np.uint64))


def test_matmul_seam_vs_oracle_odd_shape():
    import torch

    from oracle import oracle as O
    from paper_2506_02486_b200 import kernels
    rng = np.random.default_rng(9)
    a, b = rng.uniform(-1, 1, (130, 77)), rng.uniform(-1, 1, (77, 201))
    c = torch.empty(130, 201, dtype=torch.float64, device="cuda")
    kernels.matmul_f64(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), c)
    assert np.array_equal(c.cpu().numpy().view(np.uint64), O.matmul_f64(a, b).view(np.uint64))


@pytest.mark.parametrize("mnk", [(128, 128, 16), (256, 384, 512), (200, 130, 66), (1024, 2048, 512),
                                 (45, 90, 45), (129, 77, 33), (1, 1, 1), (3, 5, 0),
                                 (130, 258, 34), (1000, 1002, 998), (7, 2, 2)])
def test_dgemm_accumulate_rel_l2(mnk):
    import torch

    from paper_2506_02486_b200 import gemm
    M, N, K = mnk
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.rand(M, K, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B = torch.rand(K, N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    C0 = torch.rand(M, N, dtype=torch.float64, device="cuda", generator=g)
    C = C0.clone()
    gemm.dgemm_accumulate(A, B, C)
    want = C0.cpu().numpy() + A.cpu().numpy() @ B.cpu().numpy()
    err = np.linalg.norm(C.cpu().numpy() - want) / np.linalg.norm(want)
    assert err <= 1e-12, err


def test_dgemm_submatrix_views_and_forward():
    """Strided blocks (A[:, s*ns:(s+1)*ns]) and the fused B forwarding copy."""
    import torch

    from paper_2506_02486_b200 import gemm
    n, ns = 512, 256
    A = torch.rand(ns, n, dtype=torch.float64, device="cuda")
    B = torch.rand(ns, n, dtype=torch.float64, device="cuda")
    C = torch.zeros(ns, n, dtype=torch.float64, device="cuda")
    F = torch.full((ns, n), -1.0, dtype=torch.float64, device="cuda")
    gemm.dgemm_accumulate(A[:, ns:2 * ns], B, C, fwd=F)
    torch.cuda.synchronize()
    assert torch.equal(F, B)
    want = A[:, ns:2 * ns].cpu().numpy() @ B.cpu().numpy()
    err = np.linalg.norm(C.cpu().numpy() - want) / np.linalg.norm(want)
    assert err <= 1e-12


def test_dgemm_unaligned_views():
    """Operands that start at an odd element offset (8-byte aligned only) and
    odd leading dimensions take the 8-byte-copy variant of the same kernel."""
    import torch

    from paper_2506_02486_b200 import gemm
    g = torch.Generator(device="cuda").manual_seed(11)
    big = torch.rand(300, 301, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    A = big[1:130, 3:70]          # 129 x 67, ld 301, base offset odd
    B = big[5:72, 101:240]        # 67 x 139
    C0 = torch.rand(129, 139, dtype=torch.float64, device="cuda", generator=g)
    C = C0.clone()
    gemm.dgemm_accumulate(A, B, C)
    want = C0.cpu().numpy() + A.cpu().numpy() @ B.cpu().numpy()
    err = np.linalg.norm(C.cpu().numpy() - want) / np.linalg.norm(want)
    assert err <= 1e-12, err

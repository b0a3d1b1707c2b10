"""The reference-side binding shown in INTEGRATION.md ("ctypes stub a maintainer
would add to the reference") runs as written: grouped f32 GEMM through armt_gemm,
checked against NumPy on the reference's (G, m, k) @ (G, k, n) layout."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_05229_b200._lib import LIB_PATH, ArmtGemmArgs, EPI_STORE, F32, check, load  # noqa: E402

_lib = load(LIB_PATH)


def grouped_gemm_b200(a3: np.ndarray, b3: np.ndarray) -> np.ndarray:
    """INTEGRATION.md §2 stub, verbatim apart from the library path."""
    A = torch.from_numpy(np.ascontiguousarray(a3, np.float32)).cuda()
    Bt = torch.from_numpy(np.ascontiguousarray(b3.transpose(0, 2, 1), np.float32)).cuda()
    G, m, k = A.shape
    n = Bt.shape[1]
    C = torch.empty(G, m, n, device="cuda")
    args = ArmtGemmArgs(G=G, M=m, N=n, K=k, ab_dtype=F32, A=A.data_ptr(), lda=k, a_stride=m * k,
                        B=Bt.data_ptr(), ldb=k, b_stride=n * k, C=C.data_ptr(), ldc=n,
                        c_stride=m * n, c_dtype=F32, epilogue=EPI_STORE)
    for g in range(G):
        args.a_slot[g] = args.b_index[g] = args.c_slot[g] = g
    check(_lib.armt_gemm(ctypes.byref(args), torch.cuda.current_stream().cuda_stream), "armt_gemm")
    return C.cpu().numpy()


@pytest.mark.parametrize("G,m,k,n", [(3, 80, 128, 384), (1, 7, 64, 33), (16, 128, 256, 96)])
def test_integration_stub_matches_numpy(G, m, k, n):
    rng = np.random.default_rng(G * 1000 + m)
    a3 = rng.standard_normal((G, m, k)).astype(np.float32)
    b3 = rng.standard_normal((G, k, n)).astype(np.float32)
    got = grouped_gemm_b200(a3, b3)
    want = np.einsum("gmk,gkn->gmn", a3.astype(np.float64), b3.astype(np.float64))
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5

"""Host-side check of the GEMV weight layout (decode.frag16) against an
emulation of what the megakernel's tensor-core consumer does with it
(body_gemv in csrc/kernels/megakernel.cu): per tile, lane (g, q) loads 16 B of
A fragment and 16 B of activations x[b][32p + 8q ...], and the m16n8k16 MMA
sums A[m][kappa] * B[kappa][n] over its 16 internal k slots.  The emulated
products must equal W @ x exactly (integer-valued data, no rounding)."""

import numpy as np
import pytest
import torch

from paper_2604_13327_b200.decode import frag16


def emulate(tiled, x, N, K):
    """D[row][b] from the tiled weights the way the kernel indexes them."""
    nb = x.shape[0]
    tiles = tiled.reshape(N // 16, K // 16, 32, 8)
    D = np.zeros((N, nb))
    for t in range(N // 16):
        for j in range(K // 16):
            p, e = divmod(j, 2)
            A = np.zeros((16, 16))
            B = np.zeros((16, 8))
            for lane in range(32):
                g, q = divmod(lane, 4)
                a = tiles[t, j, lane]
                A[g, 2 * q:2 * q + 2] = a[0:2]
                A[g + 8, 2 * q:2 * q + 2] = a[2:4]
                A[g, 2 * q + 8:2 * q + 10] = a[4:6]
                A[g + 8, 2 * q + 8:2 * q + 10] = a[6:8]
                if g < nb:
                    xv = x[g, 32 * p + 8 * q:32 * p + 8 * q + 8]
                    b0, b1 = (xv[0:2], xv[2:4]) if e == 0 else (xv[4:6], xv[6:8])
                    B[2 * q:2 * q + 2, g] = b0
                    B[2 * q + 8:2 * q + 10, g] = b1
            D[16 * t:16 * t + 16] += (A @ B)[:, :nb]
    return D


@pytest.mark.parametrize("N,K,nb", [(16, 32, 1), (32, 64, 1), (48, 96, 3), (32, 128, 8)])
def test_frag16_matches_dense_product(N, K, nb):
    g = torch.Generator().manual_seed(N * K + nb)
    W = torch.randint(-4, 5, (N, K), generator=g).to(torch.bfloat16)
    x = torch.randint(-4, 5, (nb, K), generator=g).float().numpy()
    tiled = frag16(W).float().numpy()
    got = emulate(tiled, x, N, K)
    want = W.float().numpy() @ x.T
    assert np.array_equal(got, want)


def test_frag16_row_ranges_are_contiguous():
    """A task streams rows [r0, r1) (multiples of 16) as one byte range."""
    N, K = 64, 64
    W = torch.arange(N * K, dtype=torch.float32).reshape(N, K)
    T = frag16(W)
    for r0 in range(0, N, 16):
        block = T[r0:r0 + 16].flatten()
        assert sorted(block.tolist()) == sorted(W[r0:r0 + 16].flatten().tolist())

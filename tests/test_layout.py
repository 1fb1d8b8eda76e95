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


def test_tensor_core_weight_layout_matches_kernel_offsets():
    """batch.tc_pack puts W[r][k] where body_gemv_tc's descriptors read it: piece, 128-row
    block, 4 KB k step, then 8-row group (256 B), k half (128 B), row (16 B), k (2 B)."""
    import random

    import torch

    from paper_2604_13327_b200.batch import tc_pack

    N, K, kp = 256, 384, 128
    w = torch.arange(N * K, dtype=torch.float32).reshape(N, K)
    p = tc_pack(w, kp)
    nblk = N // 128
    rnd = random.Random(0)
    for _ in range(2000):
        r, k = rnd.randrange(N), rnd.randrange(K)
        piece, kk, blk, rr = k // kp, k % kp, r // 128, r % 128
        byte = ((piece * nblk + blk) * (kp * 256) + (kk // 16) * 4096 + (rr // 8) * 256 + ((kk % 16) // 8) * 128
                + (rr % 8) * 16 + (k % 8) * 2)
        assert p[byte // 2] == w[r, k]


def test_tensor_core_activation_layout_roundtrip():
    """xb_unpack inverts the operand layout of ops.cuh xb_offset (restated here)."""
    import torch

    from paper_2604_13327_b200.batch import tc_npad, xb_unpack

    b, K, kp = 5, 256, 128
    npad = tc_npad(b)

    def xb_offset(n, k):
        piece, kk = k // kp, k % kp
        return piece * npad * kp + (kk >> 4) * (npad * 16) + (n >> 3) * 128 + ((kk >> 3) & 1) * 64 + (n & 7) * 8 + (k & 7)

    x = torch.randn(b, K)
    buf = torch.zeros(npad * K)
    for n in range(b):
        for k in range(K):
            buf[xb_offset(n, k)] = x[n, k]
    assert torch.equal(xb_unpack(buf, b, K, npad, kp), x)


def test_batched_attention_grid_is_covered_by_power_of_two_samples():
    """The flat attention grid b*kv*max(1, min(ceil(s/64), cap, budget // b)) is not
    monotone in b (b=17, s=100: 272 tasks; b=32: 256), so the runtime takes the first
    covering sample whose grids also cover (runtime.cu et_step); with power-of-two batch
    samples up to 64 one always exists."""
    from paper_2604_13327_b200.batch import attn_budget
    from paper_2604_13327_b200.decode import LLAMA3_8B

    cap, bud = 18, attn_budget(LLAMA3_8B, 148)

    def tasks(b, s):
        return b * LLAMA3_8B.kv_heads * max(1, min(min((s + 63) // 64, cap), bud // b))

    for s in (1, 100, 1024, 8192):
        for b in range(1, 65):
            samples = [1 << i for i in range(7) if (1 << i) >= b]
            assert any(tasks(b, s) <= tasks(x, s) for x in samples), (b, s)


def test_moe_layout_rejects_expert_row_splits_wider_than_the_accumulators():
    """body_moe_expert holds gate / up accumulators for 8 tokens plus the activations in
    2048 floats: at most 96 rows per expert row split (the runtime rejects wider ones at
    bind time too; row_splits=6 at Qwen3's 768 rows had overrun it)."""
    import dataclasses

    from paper_2604_13327_b200.moe import QWEN3_30B_A3B, moe_layout

    moe_layout(QWEN3_30B_A3B, 148, (1024,), "static")  # 64 rows per split
    moe_layout(dataclasses.replace(QWEN3_30B_A3B, row_splits=8), 148, (1024,), "static")  # 96
    with pytest.raises(AssertionError):
        moe_layout(dataclasses.replace(QWEN3_30B_A3B, row_splits=6), 148, (1024,), "static")  # 128

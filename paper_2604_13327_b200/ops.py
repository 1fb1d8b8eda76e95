"""Host-side builders for `et_op` records (include/et_runtime.h).

Each record binds one call of a lowered graph to a tile operation of the
megakernel; the parameter layout per kind is documented in
csrc/kernels/ops.cuh.  Records are packed with ctypes and handed to
`Executor.bind_ops` as bytes.
"""

import ctypes

from . import etsim

OP_NONE = 0
OP_SPLITK_PARTIAL = 1
OP_SPLITK_FINAL = 2
OP_GEMV = 3
OP_ATTN_SPLIT = 4
OP_ATTN_MERGE = 5
OP_MOE_ROUTE = 6
OP_MOE_EXPERT = 7
OP_ALLREDUCE = 8
OP_MOE_GROUP = 9
OP_MOE_COMBINE = 10
OP_ARGMAX = 11
OP_EMBED = 12
OP_GEMV_TC = 13
OP_NORM = 14
OP_REDUCE = 15
OP_COPY = 16

EPI_F32, EPI_BF16, EPI_RESID, EPI_SILU_MUL, EPI_QKV_ROPE, EPI_ADD = range(6)

GEMV_ARGMAX = 32  # GEMV flags bit 5: the lm_head folds its rows into the step's greedy argmax word


def argmax_token(word):
    """Token id of a greedy argmax word (ordered float bits << 32 | ~row, megakernel.cu argmax_key)."""
    return (~int(word)) & 0xFFFFFFFF


class EtOp(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("i", ctypes.c_int32 * 14),
        ("f", ctypes.c_float * 4),
        ("p", ctypes.c_uint64 * 12),
    ]


assert ctypes.sizeof(EtOp) == etsim.OP_BYTES, "et_op layout mismatch with the native library"


def make_op(kind, i=(), f=(), p=(), flags=0):
    op = EtOp()
    op.kind = kind
    op.flags = flags
    for k, v in enumerate(i):
        op.i[k] = int(v)
    for k, v in enumerate(f):
        op.f[k] = float(v)
    for k, v in enumerate(p):
        op.p[k] = int(v) if v is not None else 0
    return op


def pack(ops):
    """Concatenate a list of EtOp (None = synthetic body) into bytes."""
    buf = bytearray()
    for op in ops:
        buf += bytes(op if op is not None else EtOp())
    return bytes(buf)


def ptr(t):
    """Device address of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())

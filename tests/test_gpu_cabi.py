"""The C ABI driven directly (ctypes, no pybind, no torch tensors on the path):
et_create -> et_upload_graph -> et_upload_static -> et_bind_ops -> et_step ->
et_read_counters / et_read_trace -> et_destroy, on the paper's split-K row sum
(section 2.2): partial[r][p] = sum of data[r][p][:], final[r] = sum_p partial[r][p],
with the Event Tensor E[r] (count P) between the two calls.  This is what the
reference-side binding in INTEGRATION.md calls.  Also: a rejected op table leaves
the runtime unbound, and a device error of an asynchronous step is not lost when
later steps are launched before it is collected (sticky status)."""
import ctypes

import numpy as np
import pytest

import paper_2604_13327_b200 as pkg
from paper_2604_13327_b200.ops import OP_MOE_GROUP, OP_SPLITK_FINAL, OP_SPLITK_PARTIAL, EtOp

pytestmark = pytest.mark.gpu

I32P = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)


class Config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("num_workers", ctypes.c_int32), ("record_trace", ctypes.c_int32),
                ("enable_prefetch", ctypes.c_int32), ("watchdog_ns", ctypes.c_int64), ("tick_ns", ctypes.c_int64),
                ("step_limit", ctypes.c_int64), ("max_batch", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("l2_prefetch_bytes", ctypes.c_int64)]


class GraphDesc(ctypes.Structure):
    _fields_ = [("num_symbols", ctypes.c_int32), ("num_calls", ctypes.c_int32), ("call_rank", I32P),
                ("call_extent_from", I32P), ("grid_code_off", I32P), ("code_op", I32P), ("code_arg", I64P),
                ("code_len", ctypes.c_int32), ("num_runtime_tensors", ctypes.c_int32), ("runtime_capacity", I64P),
                ("runtime_len_off", I32P)]


class SampleDesc(ctypes.Structure):
    _fields_ = [("binding", I64P), ("call_extents", I32P), ("num_queues", ctypes.c_int32),
                ("has_dma", ctypes.c_int32), ("queue_off", I32P), ("num_slots", ctypes.c_int32),
                ("slot_task", I32P), ("slot_call", I32P), ("slot_flat", I32P), ("slot_duration", I32P),
                ("wait_off", I32P), ("waits", I32P), ("notify_off", I32P), ("notifies", I32P),
                ("num_counters", ctypes.c_int32), ("initial_counts", I32P), ("counter_dd", I32P)]


class StepInfo(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("sample_index", ctypes.c_int32), ("worker", ctypes.c_int32),
                ("slot", ctypes.c_int32), ("counter", ctypes.c_int32), ("value", ctypes.c_int32),
                ("tasks_executed", ctypes.c_int64), ("noop_tasks", ctypes.c_int64), ("pushes", ctypes.c_int64),
                ("pops", ctypes.c_int64), ("kernel_ms", ctypes.c_float), ("step_id", ctypes.c_int32)]


class TraceRec(ctypes.Structure):
    _fields_ = [("t_push", ctypes.c_int64), ("t_begin", ctypes.c_int64), ("t_wait_end", ctypes.c_int64),
                ("t_prologue", ctypes.c_int64), ("t_exec_end", ctypes.c_int64), ("t_notify_end", ctypes.c_int64),
                ("worker", ctypes.c_int32), ("flags", ctypes.c_int32), ("task", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


def arr(ctype, values):
    a = (ctype * max(1, len(values)))(*values)
    return ctypes.cast(a, ctypes.POINTER(ctype)), a


R, P, L, W = 3, 4, 1000, 2  # rows, parts, elements per part, workers


@pytest.fixture(scope="module")
def lib():
    lib = ctypes.CDLL(pkg.LIBRARY_PATH)
    lib.et_last_error.restype = ctypes.c_char_p
    return lib


def upload(lib, rt, final_count=P):
    keep = []

    def a(ctype, v):
        p, o = arr(ctype, v)
        keep.append(o)
        return p

    g = GraphDesc(num_symbols=0, num_calls=2, call_rank=a(ctypes.c_int32, [2, 1]),
                  call_extent_from=a(ctypes.c_int32, [-1, -1]),
                  grid_code_off=a(ctypes.c_int32, [0, 1, 2, 2, 2, 3, 3, 3, 3]),
                  code_op=a(ctypes.c_int32, [0, 0, 0]), code_arg=a(ctypes.c_int64, [R, P, R]), code_len=3,
                  num_runtime_tensors=0, runtime_capacity=a(ctypes.c_int64, []), runtime_len_off=a(ctypes.c_int32, [0]))
    assert lib.et_upload_graph(rt, ctypes.byref(g)) == 0, lib.et_last_error(rt)
    # tasks in program order (partials row-major, then finals), dealt round-robin (ref sched_static.cpp:80-97)
    tasks = [(0, r * P + p, [], [r]) for r in range(R) for p in range(P)] + [(1, r, [r], []) for r in range(R)]
    queues = [[t for i, t in enumerate(tasks) if i % W == q] for q in range(W)]
    ids = [[i for i in range(len(tasks)) if i % W == q] for q in range(W)]
    slots = [t for q in queues for t in q]
    qoff = [0, len(queues[0]), len(slots)]
    woff, noff, waits, nots = [0], [0], [], []
    for call, flat, w, n in slots:
        waits += w
        nots += n
        woff.append(len(waits))
        noff.append(len(nots))
    s = SampleDesc(binding=a(ctypes.c_int64, []), call_extents=a(ctypes.c_int32, [R, P, 1, 1, R, 1, 1, 1]),
                   num_queues=W, has_dma=0, queue_off=a(ctypes.c_int32, qoff), num_slots=len(slots),
                   slot_task=a(ctypes.c_int32, [i for q in ids for i in q]),
                   slot_call=a(ctypes.c_int32, [t[0] for t in slots]),
                   slot_flat=a(ctypes.c_int32, [t[1] for t in slots]), slot_duration=None,
                   wait_off=a(ctypes.c_int32, woff), waits=a(ctypes.c_int32, waits),
                   notify_off=a(ctypes.c_int32, noff), notifies=a(ctypes.c_int32, nots), num_counters=R,
                   initial_counts=a(ctypes.c_int32, [final_count] * R), counter_dd=None)
    assert lib.et_upload_static(rt, ctypes.byref(s), 1) == 0, lib.et_last_error(rt)
    return len(slots)


def bind(lib, rt, dev_data, dev_part, dev_out, kind0=OP_SPLITK_PARTIAL):
    ops = (EtOp * 2)()
    ops[0].kind, ops[0].i[0], ops[0].i[1] = kind0, L, P
    ops[0].p[0], ops[0].p[1] = dev_data, dev_part
    ops[1].kind, ops[1].i[1] = OP_SPLITK_FINAL, P
    ops[1].p[1], ops[1].p[2] = dev_part, dev_out
    return lib.et_bind_ops(rt, ops, 2)


def test_cabi_splitk_rowsum_end_to_end(lib):
    import torch  # device memory only

    cfg = Config(device=0, num_workers=W, record_trace=1, enable_prefetch=1, watchdog_ns=2_000_000_000, max_batch=1,
                 l2_prefetch_bytes=-1)
    rt = ctypes.c_void_p()
    assert lib.et_create(ctypes.byref(cfg), ctypes.byref(rt)) == 0
    nslots = upload(lib, rt)
    rng = np.random.default_rng(0)
    data = rng.integers(-1000, 1000, size=(R, P, L), dtype=np.int32)
    d_data = torch.from_numpy(data).cuda()
    d_part = torch.zeros(R * P, dtype=torch.int32, device="cuda")
    d_out = torch.zeros(R, dtype=torch.int32, device="cuda")
    assert bind(lib, rt, d_data.data_ptr(), d_part.data_ptr(), d_out.data_ptr()) == 0, lib.et_last_error(rt)
    info = StepInfo()
    for _ in range(3):  # the two counter parities alternate between steps
        assert lib.et_step(rt, None, 0, None, 1, ctypes.byref(info)) == 0, lib.et_last_error(rt)
        assert info.status == 0 and info.tasks_executed == R * P + R and info.noop_tasks == 0
        assert d_out.cpu().numpy().tolist() == data.sum(axis=(1, 2)).tolist()
        assert d_part.cpu().numpy().reshape(R, P).tolist() == data.sum(axis=2).tolist()
        cnt = (ctypes.c_int64 * R)()
        assert lib.et_read_counters(rt, cnt, R) == 0 and list(cnt) == [0] * R
        recs, n = (TraceRec * nslots)(), ctypes.c_int64(nslots)
        assert lib.et_read_trace(rt, recs, ctypes.byref(n)) == 0 and n.value == nslots
        for r in recs:  # each final ran after its row's partials notified (trace order)
            assert r.t_begin <= r.t_wait_end <= r.t_exec_end <= r.t_notify_end
    assert lib.et_destroy(rt) == 0


def test_cabi_rejected_op_table_and_sticky_device_error(lib):
    import torch

    cfg = Config(device=0, num_workers=W, record_trace=0, enable_prefetch=1, watchdog_ns=50_000_000, max_batch=1,
                 l2_prefetch_bytes=-1)
    rt = ctypes.c_void_p()
    assert lib.et_create(ctypes.byref(cfg), ctypes.byref(rt)) == 0
    upload(lib, rt, final_count=P + 1)  # one notify short: every final task deadlocks
    d_data = torch.ones(R * P * L, dtype=torch.int32, device="cuda")
    d_part = torch.zeros(R * P, dtype=torch.int32, device="cuda")
    d_out = torch.zeros(R, dtype=torch.int32, device="cuda")
    # an op kind without a device body is rejected, and leaves nothing bound
    assert bind(lib, rt, d_data.data_ptr(), d_part.data_ptr(), d_out.data_ptr(), kind0=OP_MOE_GROUP) == 1
    assert lib.et_step(rt, None, 0, None, 1, None) == 1 and b"not bound" in lib.et_last_error(rt)
    assert bind(lib, rt, d_data.data_ptr(), d_part.data_ptr(), d_out.data_ptr()) == 0
    # three asynchronous steps; the first deadlocks -- the error survives the later launches
    for _ in range(3):
        assert lib.et_step(rt, None, 0, None, 0, None) == 0
    info = StepInfo()
    assert lib.et_sync(rt, ctypes.byref(info)) == 3  # ET_ERR_DEADLOCK
    assert info.status == 3 and 0 <= info.counter < R
    # collected: the runtime is usable again once the program is fixed
    upload(lib, rt)
    assert lib.et_step(rt, None, 0, None, 1, ctypes.byref(info)) == 0, lib.et_last_error(rt)
    assert d_out.cpu().tolist() == [P * L] * R
    assert lib.et_destroy(rt) == 0

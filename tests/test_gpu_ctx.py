"""The context ABI: da_ctx_create/da_ctx_destroy with library-owned
streams and an NCCL communicator bound at run time; at world 1 every collective
is the identity (one GPU per gpurun box)."""

import ctypes

import pytest
import torch

from paper_1509_05194_b200 import _native

pytestmark = pytest.mark.gpu

N = _native.native


def _ctx():
    dev = (ctypes.c_int * 1)(0)
    h = ctypes.c_void_p()
    N.da_ctx_create(1, ctypes.cast(dev, ctypes.c_void_p), ctypes.byref(h))
    return h


def test_ctx_nccl_world1():
    h = _ctx()
    s = ctypes.c_void_p()
    N.da_ctx_stream(h, 0, ctypes.byref(s))
    assert s.value
    uid = ctypes.create_string_buffer(128)
    N.da_nccl_unique_id(uid)
    N.da_ctx_nccl_init(h, 0, 1, uid)
    buf = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.5 - 3.0
    ref = buf.clone()
    torch.cuda.synchronize()
    N.da_ctx_allreduce_f64(h, buf.data_ptr(), buf.numel(), None)
    cnt = torch.arange(7, dtype=torch.int32, device="cuda")
    got = torch.full((7,), -1, dtype=torch.int32, device="cuda")
    N.da_ctx_allgather_i32(h, cnt.data_ptr(), got.data_ptr(), 7, None)
    recv = torch.full((5,), 9.0, dtype=torch.float64, device="cuda")
    N.da_ctx_shift_f64(h, buf.data_ptr(), recv.data_ptr(), 5, None)   # rank 0 of 1: no peer either side
    N.da_ctx_destroy(h)                                                 # synchronizes the context's stream
    assert torch.equal(buf, ref)
    assert torch.equal(got, cnt)
    assert torch.equal(recv, torch.full((5,), 9.0, dtype=torch.float64, device="cuda"))


def test_ctx_errors():
    h = _ctx()
    buf = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="no communicator"):
        N.da_ctx_allreduce_f64(h, buf.data_ptr(), 4, None)
    s = ctypes.c_void_p()
    with pytest.raises(ValueError, match="bad index"):
        N.da_ctx_stream(h, 3, ctypes.byref(s))
    N.da_ctx_destroy(h)
    bad = (ctypes.c_int * 1)(torch.cuda.device_count())
    with pytest.raises(ValueError, match="ctx_create"):
        N.da_ctx_create(1, ctypes.cast(bad, ctypes.c_void_p), ctypes.byref(ctypes.c_void_p()))

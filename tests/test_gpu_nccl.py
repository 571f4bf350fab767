"""Native NCCL transport of the partitioned factorization (csrc/nccl_exchange.cpp)
on the one GPU a test box has: a single-rank communicator, the exchange function
called as the library calls it (all-reduces on device buffers, on a stream). The
point-to-point messages need two GPUs and are covered by construction only:
the schedule they follow is tested over gloo (tests/test_partition.py) and over
the in-process loopback (tests/test_gpu_partition.py)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nccl_exchange_single_rank():
    import torch

    from paper_2503_08343_b200 import _capi
    from paper_2503_08343_b200.partition import (MSG_ALLREDUCE_MIN_I32, MSG_ALLREDUCE_SUM_F64,
                                                 NcclExchange)
    torch.cuda.set_device(0)
    ex = NcclExchange(nranks=1, rank=0)
    try:
        x = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.5
        st = torch.tensor([7, -3, 11], dtype=torch.int32, device="cuda")
        ref_x, ref_st = x.clone(), st.clone()
        msgs = (_capi.Msg * 2)()
        msgs[0] = _capi.Msg(MSG_ALLREDUCE_SUM_F64, -1, -1, -1, x.data_ptr(), x.numel())
        msgs[1] = _capi.Msg(MSG_ALLREDUCE_MIN_I32, -1, -1, -1, st.data_ptr(), st.numel())
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        rc = ex.fn(ex.ctx, msgs, 2, C.c_void_p(stream.cuda_stream))
        assert rc == 0
        stream.synchronize()
        assert torch.equal(x, ref_x) and torch.equal(st, ref_st)  # one rank: identity
    finally:
        ex.close()

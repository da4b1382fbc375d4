"""The kernel-lane binding of INTEGRATION.md, exactly as a reference maintainer
would add it (raw ctypes on libcorrvol_b200.so, numpy in / numpy out, the
`_ckernels.pyx` lane contract), checked bit for bit against the golden lane
vectors the reference produced (tests/golden/make_golden.py)."""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2505_16942_b200 import _build

pytestmark = pytest.mark.gpu

_p, _i32, _i64 = C.c_void_p, C.c_int32, C.c_int64
STRICT = 1


@pytest.fixture(scope="module")
def lane(cuda):
    lib = C.CDLL(str(_build.LIB))
    lib.cvb_corr_pairs.argtypes = [_p, _i64, _p, _i64, _i32, _p, _i32, _p]
    lib.cvb_corr_gather.argtypes = [_p, _i64, _p, _i64, _i32, _p, _p, _p, _i32, _p]
    lib.cvb_block_mmm.argtypes = [_p, _p, _i64, _i32, _i32, _i32, _p, _i32, _p]
    lib.cvb_last_error.restype = C.c_char_p

    def check(status):
        if status:
            raise (ValueError if status == 1 else RuntimeError)(lib.cvb_last_error().decode())

    def dev(a, dtype=torch.float32):
        return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)

    stream = lambda: torch.cuda.current_stream().cuda_stream

    def corr_pairs(a, b):
        if a.shape[1] != b.shape[1]:
            raise ValueError(f"channel counts differ: {a.shape[1]} vs {b.shape[1]}")
        ta, tb = dev(a), dev(b)
        out = torch.empty((a.shape[0], b.shape[0]), device="cuda")
        check(lib.cvb_corr_pairs(ta.data_ptr(), a.shape[0], tb.data_ptr(), b.shape[0],
                                 a.shape[1], out.data_ptr(), STRICT, stream()))
        return out.cpu().numpy()

    def corr_gather(f1, f2, idx, valid):
        t1, t2 = dev(f1), dev(f2)
        ti, tv = dev(idx, torch.int64), dev(valid, torch.uint8)
        out = torch.empty(f1.shape[0], device="cuda")
        check(lib.cvb_corr_gather(t1.data_ptr(), f1.shape[0], t2.data_ptr(), f2.shape[0],
                                  f1.shape[1], ti.data_ptr(), tv.data_ptr(), out.data_ptr(),
                                  STRICT, stream()))
        return out.cpu().numpy()

    def block_mmm(at, bt):
        k, n, d = at.shape
        ta, tb = dev(at), dev(bt)
        out = torch.empty((k, n, bt.shape[1]), device="cuda")
        check(lib.cvb_block_mmm(ta.data_ptr(), tb.data_ptr(), k, n, bt.shape[1], d,
                                out.data_ptr(), STRICT, stream()))
        return out.cpu().numpy()

    return corr_pairs, corr_gather, block_mmm


def test_integration_lane_bit_exact(golden, lane):
    corr_pairs, corr_gather, block_mmm = lane
    assert np.array_equal(corr_pairs(golden["lane/a"], golden["lane/b"]), golden["lane/pairs"])
    assert np.array_equal(corr_gather(golden["lane/g_f1"], golden["lane/g_f2"],
                                      golden["lane/g_idx"], golden["lane/g_valid"]),
                          golden["lane/gather"])
    assert np.array_equal(block_mmm(golden["lane/at"], golden["lane/bt"]), golden["lane/mmm"])


def test_integration_lane_errors(lane):
    corr_pairs, _, _ = lane
    with pytest.raises(ValueError):
        corr_pairs(np.zeros((2, 3), np.float32), np.zeros((2, 4), np.float32))

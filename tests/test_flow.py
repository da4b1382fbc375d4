"""Cascaded-init flow resample (flowio.py:151-199) on the GPU: bit-identical
to the reference; the reference's own known answers (test_flowio.py:218-275)."""

import numpy as np
import pytest
import torch

import paper_2505_16942_b200 as cvb
from oracle import import_reference

pytestmark = pytest.mark.gpu


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)


@pytest.mark.parametrize("shape,scale", [((37, 53), 0.5), ((20, 31), 2.0), ((9, 14), 1.0),
                                         ((64, 48), 0.37), ((7, 5), 3.3), ((1, 9), 0.5),
                                         ((135, 240), 0.5)])
def test_resample_bit_identical_to_reference(cuda, shape, scale):
    ref = import_reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from corrvol.flowio import resample_flow as ref_resample
    rng = np.random.default_rng(sum(shape))
    f = (rng.standard_normal(shape + (2,)) * 7).astype(np.float32)
    want = ref_resample(ref.FlowField(vectors=f.copy()), scale).vectors
    got = cvb.resample_flow(_t(f, cuda), scale).cpu().numpy()
    assert got.shape == want.shape and np.array_equal(got, want)


def test_resample_known_answers(cuda):
    f = np.full((6, 10, 2), 3.0, np.float32)
    assert np.array_equal(cvb.resample_flow(_t(f, cuda), 1.0).cpu().numpy(), f)
    half = cvb.cascaded_init(_t(f, cuda)).cpu().numpy()
    assert half.shape == (3, 5, 2) and np.all(half == 1.5)  # constant field, halved
    odd = cvb.resample_flow(_t(np.zeros((5, 7, 2)), cuda), 0.5)
    assert tuple(odd.shape) == (3, 4, 2)  # round half up (test_flowio.py:272-275)
    with pytest.raises(ValueError):
        cvb.resample_flow(_t(f, cuda), 0.05)
    with pytest.raises(ValueError):
        cvb.resample_flow(_t(f, cuda), -1.0)

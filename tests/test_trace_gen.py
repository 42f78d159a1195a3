"""The skewed routing generator (host C++, libmoesim_b200.so) reproduces the
reference generator (trace.cpp:174-259, verbatim build) bit for bit."""
import numpy as np
import pytest

from oracle import native as N
from paper_2303_06182_b200.traces import skewed_routing


@pytest.mark.skipif(not N.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("E,k,B,S,skew,pers,frac,seed", [(128, 2, 5, 300, 1.2, 0.9, 1.0, 42),
                                                        (16, 1, 7, 50, 0.0, 0.0, 0.5, 1),
                                                        (512, 2, 3, 1000, 2.0, 0.5, 0.25, 2303)])
def test_generator_matches_reference(E, k, B, S, skew, pers, frac, seed):
    ex, w = skewed_routing(E, k, B, S, skew, pers, frac, seed)
    rex, rw = N.ref_gen_synthetic_trace(E, k, B, S, skew, pers, frac, seed)
    assert (ex == rex).all()
    assert (w == rw).all()


def test_generator_errors_and_skew():
    with pytest.raises(ValueError, match="not enough active experts for top-k"):
        skewed_routing(4, 3, 1, 10, 1.0, 0.5, 0.5, 0)
    ex, w = skewed_routing(64, 2, 1, 4000, 1.2, 0.9, 1.0, 3)
    cnt = np.bincount(ex.reshape(-1), minlength=64)
    assert cnt.max() > 8 * np.median(cnt)  # Zipf skew
    assert (ex[..., 0] != ex[..., 1]).all()
    assert np.abs(w.sum(-1) - 1).max() < 1e-12

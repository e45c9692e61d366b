"""FourierTransformer surface that needs no GPU (reference tests/test_estimator.py)."""

import numpy as np
import pytest
from sklearn.base import clone
from sklearn.exceptions import NotFittedError

from paper_2203_09384_b200 import FourierTransformer, InvalidLengthError, ShapeError, UnsupportedLengthError


def test_params_clone_and_fit_plans():
    est = FourierTransformer(direction="inverse", algorithm="split", precision="double")
    assert est.get_params() == {"direction": "inverse", "algorithm": "split", "precision": "double"}
    assert clone(est).get_params() == est.get_params()
    est.fit(np.ones((2, 64)))
    assert est.plan_.length == 64 and est.plan_.direction.value == "inverse"
    assert est.inverse_plan_.direction.value == "forward"
    assert est.n_features_in_ == 64


def test_fit_errors():
    with pytest.raises(NotFittedError):
        FourierTransformer().transform(np.ones((1, 8)))
    with pytest.raises(ShapeError):
        FourierTransformer().fit(np.ones(64, np.complex64))
    with pytest.raises(UnsupportedLengthError):
        FourierTransformer().fit(np.ones((2, 4096)))
    with pytest.raises(InvalidLengthError):
        FourierTransformer().fit(np.ones((2, 12)))
    with pytest.raises(InvalidLengthError):
        FourierTransformer().fit(np.ones((0, 8)))


def test_validation_helpers_reference_semantics():
    """validation.py:10-57: shape -> emptiness -> dtype -> finiteness, any strides."""
    import numpy as np
    import pytest

    from paper_2203_09384_b200 import DomainError, InvalidLengthError, ShapeError
    from paper_2203_09384_b200.validation import COMPLEX_DTYPE, as_signal, check_same_length, check_signal_matrix

    x = (np.arange(16) + 1j).astype(np.complex128)
    s = as_signal(x[::2])  # strided input
    assert s.dtype == COMPLEX_DTYPE == np.complex64 and s.shape == (8,)
    assert as_signal(x, dtype=np.complex128) is x  # no copy when already the target dtype
    bad = x.copy()
    bad[3] = complex(0, np.inf)
    with pytest.raises(DomainError):
        as_signal(bad)
    with pytest.raises(ShapeError):
        as_signal(np.ones((2, 2)))
    with pytest.raises(InvalidLengthError):
        as_signal(np.array([]))
    with pytest.raises(DomainError):
        as_signal(np.array(["a", "b"]))
    with pytest.raises(ShapeError):
        check_same_length(np.ones(3), np.ones(4))
    with pytest.raises(ShapeError):
        check_signal_matrix(np.ones(8))
    with pytest.raises(InvalidLengthError):
        check_signal_matrix(np.ones((0, 8)))
    m = check_signal_matrix(np.ones((3, 8))[:, ::2])
    assert m.dtype == np.complex64 and m.shape == (3, 4)
    # the estimator's GPU route leaves value checks to the kernel and keeps reals real
    r = check_signal_matrix(np.full((2, 4), np.nan), kernel_checks=True)
    assert r.dtype == np.float64

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

"""The test-side torch checksum equals the oracle's (-m "not gpu"): the GPU
tests form table digests on the device with tests/devtools.py and compare
them with digests the oracle recorded (tests/golden/c3_i18.json)."""
import numpy as np
import torch

import oracle
from tests import devtools


def test_torch_mixsum_equals_oracle_mixsum():
    rng = np.random.default_rng(5)
    a = rng.integers(0, 1 << 30, 100003).astype(np.int32)
    a[::7] = 1 << 30
    u = rng.integers(0, 5, 100003).astype(np.uint8)
    f = rng.random(5001) * 1e3
    for arr, salt in ((a, 1), (u, 2), (f, 1)):
        assert devtools.mixsum(torch.from_numpy(arr), salt, chunk=4099) == oracle.mixsum(arr, salt)
    assert devtools.mix_digest(torch.from_numpy(a), torch.from_numpy(u)) == oracle.mix_digest(a, u)


def test_near_tie_rule():
    s = np.array([[1.0, 1.0 + 1e-12, 5.0], [2.0, 3.0, 2.0], [np.inf, np.inf, 1.0]])
    ok = devtools.near_tie_ok(s, np.array([1, 1, 0]), np.array([0, 0, 1]))
    assert list(ok) == [True, False, True]

"""Test helpers shared by the CPU and GPU suites."""

import os

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")


def load_golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not present")
    return dict(np.load(path, allow_pickle=False))


class StubSampler:
    """Injects a fixed k-set: rb_energy_forces only calls sampler.batch(P)
    (reference rbse2d.py:288)."""

    def __init__(self, modes):
        self.modes = np.asarray(modes)

    def batch(self, P):
        assert P == self.modes.shape[0]
        return self.modes



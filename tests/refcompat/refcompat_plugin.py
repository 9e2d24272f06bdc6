"""pytest plugin for the reference-suite run (tools/run_reference_tests.sh).

The reference's test_zero_mode_matches_direct_pair_evaluation
(pkg/tests/test_soewald2d.py:251-269) encodes the paper's Eq. 32 zero-mode
split, which the reference code does not implement: it
fails against the reference itself.  The drop-in follows the code, so the test
is marked as a strict expected failure here -- it must still fail."""

import pytest

KNOWN_REFERENCE_FAILURES = {
    "test_soewald2d.py::test_zero_mode_matches_direct_pair_evaluation":
        "paper Eq. 32 vs the reference code's zero-mode split: fails on the reference too",
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        key = f"{item.path.name}::{item.name}"
        if key in KNOWN_REFERENCE_FAILURES:
            item.add_marker(pytest.mark.xfail(reason=KNOWN_REFERENCE_FAILURES[key], strict=True))

"""``slabewald`` -> this drop-in: lets the reference's OWN test modules
(pkg/tests/test_soewald2d.py, test_rbse2d.py) import the reference's module
paths and run against the B200 implementation unchanged.

Test infrastructure only (tools/run_reference_tests.sh puts this directory on
PYTHONPATH); the product package is ``paper_2403_01521_b200``.
"""

import sys

import paper_2403_01521_b200 as _pk
from paper_2403_01521_b200 import *  # noqa: F401,F403  (the public API, as the reference's __init__)
from paper_2403_01521_b200 import core, ewald2d, md, rbse2d, soewald2d  # noqa: F401

from . import soe  # noqa: F401  (our soe plus the pointwise xi_soe test shim)

for _name in ("core", "ewald2d", "md", "rbse2d", "soewald2d"):
    sys.modules[f"{__name__}.{_name}"] = getattr(_pk, _name)

__all__ = list(getattr(_pk, "__all__", []))

"""Drop-in alias: ``gpp.oracle`` (``exhaustive_optimize``,
``min_inflight_search``) is the repo's test-only brute-force oracle ``oracle.brute``.

The reference ships ``gpp`` as a namespace package (pkg/pyproject.toml:6-12, no
__init__.py).  SPEC.md:483 keeps the oracle off the hot path; so does this alias —
nothing in ``paper_2406_17145_b200`` imports it.
"""
import sys as _sys

from oracle import brute as _impl

_sys.modules[__name__] = _impl

"""Drop-in alias: ``gpp.partition`` is ``paper_2406_17145_b200.partition`` (the same module object).

The reference ships ``gpp`` as a namespace package (pkg/pyproject.toml:6-12, no
__init__.py); code written against it imports this module unchanged.
"""
import sys as _sys

from paper_2406_17145_b200 import partition as _impl

_sys.modules[__name__] = _impl

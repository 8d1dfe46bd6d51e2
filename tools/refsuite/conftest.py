"""Drop-in check: the reference package's OWN unit tests (pkg/tests/test_*.py of the reference,
unmodified, copied next to this file only for the duration of a run and never committed) import
`spirk.*`; this conftest makes `spirk` resolve to the B200 package so every call in those tests goes
through the device path (numpy arrays in, numpy arrays out: INTEGRATION.md §1).

Run: python tools/refsuite/run.py <reference pkg/tests dir> (see tools/refsuite/run.py)."""

import sys

# run.py puts the repository on PYTHONPATH (this file is copied into a scratch directory)

import paper_2209_06700_b200 as _pkg  # noqa: E402
from paper_2209_06700_b200 import errors, fem, krylov, multigrid, tableau  # noqa: E402

sys.modules["spirk"] = _pkg
for _name, _mod in (("errors", errors), ("fem", fem), ("krylov", krylov), ("multigrid", multigrid),
                    ("tableau", tableau)):
    sys.modules["spirk." + _name] = _mod
    setattr(_pkg, _name, _mod)

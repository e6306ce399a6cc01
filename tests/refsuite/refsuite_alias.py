"""pytest plugin: run the REFERENCE's own test suite against this package.

Loaded with ``-p refsuite_alias`` by ``tests/test_reference_suite_gpu.py``.
At import time it makes ``import wtindex`` (and ``wtindex.<module>``) resolve
to ``paper_2505_03372_b200`` -- the drop-in claim, tested with the
reference's unmodified tests (copied by ``__graft_entry__._install_reference``
into the git-ignored ``baseline/_ref_tests``).

Two reference modules that are not part of the accelerated path are loaded
from the unmodified reference install (``baseline/_ref/wtindex``) on top of
the aliased package, exactly as the reference ships them:

* ``wtindex.oracle`` -- the reference's naive test oracle (test
  infrastructure: ``tests/helpers.py`` and the acceptance suite import it);
* ``wtindex.cli`` -- the reference's command-line driver (out of scope for
  the rebuild); running it over this package shows that a
  caller of the reference API works unchanged.

Both resolve their relative imports (``from .batch import ...``) to this
package's modules.
"""

import importlib.util
import os
import sys

ROOT = os.environ.get("WT_REPO_ROOT") or os.path.dirname(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2505_03372_b200 as _pkg  # noqa: E402
from paper_2505_03372_b200 import (alphabet, batch, bitvec, errors,  # noqa: E402
                                   rankselect, wtree)

sys.modules["wtindex"] = _pkg
for _name, _mod in (("alphabet", alphabet), ("batch", batch), ("bitvec", bitvec),
                    ("errors", errors), ("rankselect", rankselect), ("wtree", wtree)):
    sys.modules[f"wtindex.{_name}"] = _mod

_REF = os.path.join(ROOT, "baseline", "_ref", "wtindex")


def _load_reference_module(name: str):
    path = os.path.join(_REF, f"{name}.py")
    spec = importlib.util.spec_from_file_location(f"wtindex.{name}", path,
                                                  submodule_search_locations=None)
    mod = importlib.util.module_from_spec(spec)
    mod.__package__ = "wtindex"
    sys.modules[f"wtindex.{name}"] = mod
    spec.loader.exec_module(mod)
    setattr(_pkg, name, mod)
    return mod


_load_reference_module("oracle")
_load_reference_module("cli")

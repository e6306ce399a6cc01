"""Record the reference's public API surface (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_reference_api.py

Writes ``reference_api.json``: the reference package's ``__all__``
(/root/reference/pkg/src/wtindex/__init__.py:61-73) and, for every exported
class, its public methods / properties, plus the module-level names the
reference's own tests read from submodules.  ``tests/test_capi_cpu.py``
checks this package against it.
"""

import inspect
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import wtindex  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

out = {"__all__": sorted(wtindex.__all__), "classes": {}, "modules": {}}
for name in wtindex.__all__:
    obj = getattr(wtindex, name)
    if inspect.isclass(obj) and not issubclass(obj, BaseException):
        # methods / properties / classmethods (instance slots are data, not API)
        out["classes"][name] = sorted(
            m for m in dir(obj) if not m.startswith("_")
            and not inspect.ismemberdescriptor(inspect.getattr_static(obj, m)))
for mod in ("alphabet", "batch", "bitvec", "rankselect", "wtree", "errors"):
    m = __import__(f"wtindex.{mod}", fromlist=["x"])
    # what the module itself defines: functions / classes, and UPPER_CASE constants
    out["modules"][mod] = sorted(
        n for n, v in vars(m).items() if not n.startswith("_")
        and ((callable(v) and getattr(v, "__module__", None) == m.__name__) or n.isupper()))
with open(os.path.join(HERE, "reference_api.json"), "w") as f:
    json.dump(out, f, indent=1)
print(len(out["__all__"]), "names")

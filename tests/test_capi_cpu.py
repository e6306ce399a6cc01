"""CPU-side checks of the C-ABI boundary: the library loads and exports every
function include/wt_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "wt_b200.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(wt_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("wt_construct", "wt_tree_query", "wt_tree_get", "wt_tree_replicate",
                 "wt_bits_build", "wt_bits_query", "wt_tree_from_arrays"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2505_03372_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the python binding binds exactly the declared set
    assert sorted(_lib.EXPORTS) == declared_functions()


def test_abi_version_and_error_path_without_gpu():
    import paper_2505_03372_b200 as w
    from paper_2505_03372_b200 import _lib
    assert _lib.lib.wt_abi_version() == 1
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by the gpu tests")
    except ImportError:
        pass
    # no GPU: the product path must fail loudly, never fall back to the CPU
    with pytest.raises(w.DeviceError):
        w.construct(b"abracadabra")


def test_api_surface_matches_reference():
    """Every name of the reference's __all__, every public method of its
    exported classes and every name its modules define (recorded from the
    reference by tests/golden/make_reference_api.py) exists here."""
    import importlib
    import json

    import paper_2505_03372_b200 as w
    api = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_api.json")))
    assert sorted(w.__all__) == sorted(set(api["__all__"]) | {"DeviceError"})
    for name in api["__all__"]:
        assert hasattr(w, name), name
    for cls, members in api["classes"].items():
        missing = [m for m in members if not hasattr(getattr(w, cls), m)]
        assert not missing, (cls, missing)
    for mod, names in api["modules"].items():
        m = importlib.import_module(f"paper_2505_03372_b200.{mod}")
        missing = [n for n in names if not hasattr(m, n)]
        assert not missing, (mod, missing)


def test_recorded_api_is_the_reference_all():
    """The recorded list is the reference's own __all__ (parsed, not imported,
    from the unmodified install when it is present), not a hand-trimmed one."""
    import ast
    import json
    init = os.path.join(ROOT, "baseline", "_ref", "wtindex", "__init__.py")
    if not os.path.exists(init):
        pytest.skip("baseline/_ref absent")
    tree = ast.parse(open(init).read())
    ref_all = next(ast.literal_eval(n.value) for n in tree.body if isinstance(n, ast.Assign)
                   and any(getattr(t, "id", None) == "__all__" for t in n.targets))
    api = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_api.json")))
    assert sorted(ref_all) == api["__all__"]


def test_host_codes_match_oracle():
    import numpy as np
    import oracle as O
    from paper_2505_03372_b200 import create_codes
    for s in list(range(1, 600)) + [4095, 4097, 38158, 65535, 65536]:
        ct = create_codes(s)
        v, l, f = O.tree_codes(s)
        assert np.array_equal(ct.values, v) and np.array_equal(ct.lens, l) and ct.first_coded == f

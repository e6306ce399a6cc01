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


def test_api_surface_matches_reference_names():
    import paper_2505_03372_b200 as w
    ref_all = [
        "AlphabetMap", "BadMagicError", "BadVersionError", "BatchError",
        "BatchRunner", "BitArray", "BuildError", "Code", "CodeTable",
        "CorruptIndexError", "Error", "IndexFileError", "OrdinalError",
        "PositionError", "QueryBatch", "RankSelectIndex", "RankSelectParams",
        "SymbolError", "TruncatedError", "WaveletTree", "access_batch",
        "build_bit_array", "build_index", "ceil_log2", "construct",
        "construct_with_alphabet", "create_codes", "cumulative_histogram",
        "level_sizes", "load", "partial_word", "prev_pow_two", "rank_batch",
        "run_batch", "save", "select_batch", "select_in_word",
        "sort_queries_by_symbol",
    ]
    for name in ref_all:
        assert hasattr(w, name), name


def test_host_codes_match_oracle():
    import numpy as np
    import oracle as O
    from paper_2505_03372_b200 import create_codes
    for s in list(range(1, 600)) + [4095, 4097, 38158, 65535, 65536]:
        ct = create_codes(s)
        v, l, f = O.tree_codes(s)
        assert np.array_equal(ct.values, v) and np.array_equal(ct.lens, l) and ct.first_coded == f

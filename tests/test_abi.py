"""The C-ABI library loads and exports every symbol include/sae.h declares (no GPU
needed: dlopen only, no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sae.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sae_[a-z_]+)\s*\(", src)))


def test_header_declares_north_star_calls():
    fns = declared_functions()
    for f in ("sae_create", "sae_admit_batch", "sae_lookup", "sae_evict", "sae_update", "sae_stats"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    from paper_2605_18825_b200 import build as B
    path = B.build()
    L = ctypes.CDLL(path)
    for f in declared_functions():
        assert hasattr(L, f), f
    from paper_2605_18825_b200 import sae as S
    assert set(S.EXPORTS) == set(declared_functions())


def test_struct_sizes_match_header_layout():
    from paper_2605_18825_b200 import sae as S
    # sae_params: 20 doubles + 2 u32
    assert ctypes.sizeof(S.sae_params) == 20 * 8 + 8
    assert ctypes.sizeof(S.sae_batch) == 8 + 8 + 10 * 8
    assert ctypes.sizeof(S.sae_admit_out) == 6 * 8 + 8 + 2 * 8


def test_oracle_is_not_imported_by_product_package():
    pkg = os.path.join(ROOT, "paper_2605_18825_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f

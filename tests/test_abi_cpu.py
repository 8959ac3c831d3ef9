"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares; host-side grid/plan bookkeeping (no device calls)."""

import ctypes
import os
import re

from paper_2509_00642_b200 import _lib
from paper_2509_00642_b200.profiler import GridSpec, pair_list, prompts_hash, stable_text_key

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hadis_b200.h")


def declared_functions():
    text = open(HEADER, encoding="utf-8").read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hadis_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)


def test_library_pure_host_calls():
    lib = _lib.load()
    assert lib.hadis_abi_version() == 1
    assert lib.hadis_status_string(5) == b"fallback: no serveable rows"
    assert lib.hadis_hfix_shift(10_000_000) == 63 - 24
    assert lib.hadis_hfix_shift(1) == 48
    assert lib.hadis_frontier_workspace_bytes(6, 256, 1 << 20, 2048, 1 << 20) > 0
    assert lib.hadis_pareto_workspace_bytes(0) == 0


def test_grid_spec_duplicates_and_signed_zero():
    g = GridSpec.build((0.2, 0.6, 0.2, 1.0, 0.6))
    assert g.unique == (0.2, 0.6, 1.0) and g.first_pos == (0, 1, 3)
    g = GridSpec.build((-0.0, 0.25, 0.0, 0.75))
    assert g.unique == (-0.0, 0.25, 0.75) and g.first_pos == (0, 1, 3)
    g = GridSpec.build((0.5, 0.1, 0.9))
    assert g.unique == (0.1, 0.5, 0.9) and g.first_pos == (1, 0, 2)


def test_pairs_light_to_heavy():
    assert pair_list(list("abcd")) == [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def test_prompts_hash_is_order_free():
    # reference values are checked in test_table_cpu.py / test_text_cpu.py
    assert prompts_hash(["x", "y", "z"]) == prompts_hash(["z", "x", "y"])
    assert 0 <= stable_text_key("a cat") < 2 ** 63

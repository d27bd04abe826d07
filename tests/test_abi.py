"""CPU-side checks of the C-ABI boundary: the library loads and exports every symbol
include/ks.h declares; validation paths that fail before any device work."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ks.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^KS_API\s+[\w\s\*]+?\b(ks_\w+)\s*\(", txt, flags=re.M)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ["ks_sketch", "ks_tsqr", "ks_lowrank_solve", "ks_omega_export", "ks_tsqr_merge", "ks_qform",
              "ks_apply_qt", "ks_apply_q", "ks_trsolve", "ks_omega_apply", "ks_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1312_1869_b200 as ks
    if not os.path.exists(ks.library_path):
        from paper_1312_1869_b200 import build
        build.build()
    L = ctypes.CDLL(ks.library_path)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert ks.ks_version().startswith("ks-b200")


def test_sketch_descriptor_layout_matches_header():
    import paper_1312_1869_b200 as ks
    assert ctypes.sizeof(ks.SketchDesc) == 48
    assert ks.SketchDesc.seed.offset == 32 and ks.SketchDesc.omega.offset == 40


@pytest.mark.parametrize("field,value", [("n", 0), ("dim", 4), ("ell", 0.0), ("sigma2", -1.0), ("nugget", -1e-3),
                                         ("d", 0), ("kernel", 7), ("omega", 4)])
def test_workspace_query_rejects_invalid_descriptors(field, value):
    import paper_1312_1869_b200 as ks
    args = dict(n=1024, dim=2, kernel=0, sigma2=1.0, ell=0.1, nugget=0.0, d=64, seed=1, omega=0)
    args[field] = value
    with pytest.raises(ks.KsError) as e:
        ks.ks_sketch_workspace_size(args)
    assert e.value.status == 1
    assert ks.ks_last_error()


def test_unsupported_sizes_are_reported():
    import paper_1312_1869_b200 as ks
    with pytest.raises(ks.KsError) as e:
        ks.ks_sketch_workspace_size(dict(n=4096, dim=2, kernel=0, sigma2=1.0, ell=0.1, nugget=0.0, d=1024, seed=1,
                                         omega=0))
    assert e.value.status == 5
    with pytest.raises(ks.KsError) as e:
        ks.ks_sketch_workspace_size(dict(n=4096, dim=2, kernel=0, sigma2=1.0, ell=0.1, nugget=0.0, d=100, seed=1,
                                         omega=1))
    assert e.value.status == 5


def test_tsqr_topology_validation():
    import paper_1312_1869_b200 as ks
    chain = ks.ks_tsqr_workspace_size_ex(262144, 512, 8, ks.TSQR_CHAIN)
    tree = ks.ks_tsqr_workspace_size_ex(262144, 512, 8, ks.TSQR_TREE)
    assert chain > 262144 * 512 * 4 and tree == ks.ks_tsqr_workspace_size(262144, 512, 8)
    with pytest.raises(ks.KsError):
        ks.ks_tsqr_workspace_size_ex(1000, 10, 2, 7)


def test_tsqr_workspace_rejects_wide_blocks():
    import paper_1312_1869_b200 as ks
    with pytest.raises(ks.KsError) as e:
        ks.ks_tsqr_workspace_size(100, 64, 2)
    assert e.value.status == 1
    assert ks.ks_tsqr_workspace_size(262144, 512, 8) > 262144 * 512 * 4


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1312_1869_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "ks_oracle" not in txt, f

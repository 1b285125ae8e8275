"""The C-ABI library loads and exports every symbol include/nc.h declares (no compute calls; CPU-safe)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:int|void|char)\s*\*?\s*(nc_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("nc_setup", "nc_matvec", "nc_gmres", "nc_flux_or_mfpt", "nc_partition", "nc_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1906_04209_b200 import build, nc
    build.build()
    L = nc.load_library()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert b"sm_100a" in L.nc_version()


def test_binding_declares_every_symbol():
    from paper_1906_04209_b200 import nc
    assert set(declared_symbols()) == set(nc.EXPORTS)

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


def test_stats_struct_matches_header():
    """The ctypes mirror of nc_stats_t has the header's fields in the header's order."""
    import re
    from paper_1906_04209_b200 import nc
    src = open(os.path.join(ROOT, "include", "nc.h")).read()
    body = src[src.index("typedef struct nc_stats_t {"):src.index("} nc_stats_t;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for line in body.splitlines()[1:]:
        line = line.strip().rstrip(";")
        if not line:
            continue
        decl = line.split(None, 1)[1]
        for d in decl.split(","):
            names.append(d.strip().split("[")[0])
    assert names == [f for f, _ in nc.NcStats._fields_]

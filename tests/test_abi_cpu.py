"""CPU-side checks of the boundary: the C-ABI library loads, exports every symbol include/amg.h
declares, and the ctypes struct layouts match the header (no compute calls: no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "amg.h")


@pytest.fixture(scope="module")
def amg_mod():
    lib = os.path.join(ROOT, "paper_1307_6305_b200", "lib", "libamg_b200.so")
    if not os.path.exists(lib):
        subprocess.check_call(["make", "-C", ROOT, "-j4", "paper_1307_6305_b200/lib/libamg_b200.so"])
    from paper_1307_6305_b200 import amg

    amg.load()
    return amg


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(amg_\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(amg_mod):
    names = declared_functions()
    assert {"amg_setup", "amg_solve", "amg_free"} <= set(names)
    lib = amg_mod.load()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(amg_mod.EXPORTS)


def test_struct_layout_matches_header(amg_mod, tmp_path):
    c = tmp_path / "layout.c"
    c.write_text(f"""
#include <stdio.h>
#include <stddef.h>
#include "{HDR}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(amg_options), offsetof(amg_options, stream),
         offsetof(amg_options, use_graphs), sizeof(amg_info), offsetof(amg_info, grid_complexity),
         offsetof(amg_info, launches_last_solve));
  return 0;
}}
""")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-o", str(exe), str(c)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    O, I = amg_mod.amg_options, amg_mod.amg_info
    assert got == [ctypes.sizeof(O), O.stream.offset, O.use_graphs.offset, ctypes.sizeof(I),
                   I.grid_complexity.offset, I.launches_last_solve.offset]


def test_defaults_and_argument_errors(amg_mod):
    """Host-only paths: defaults, and argument validation that returns before touching the GPU."""
    o = amg_mod.amg_options_default()
    assert (o.coarsest_size, o.kappa, o.restart, o.max_iter, o.use_graphs, o.tail_nnz) == (100, 0.0, 5, 500, 1, 8192)
    lib = amg_mod.load()
    assert lib.amg_options_default(None) == amg_mod.AMG_E_ARG
    h = ctypes.c_void_p()
    # NULL arrays / bad degree / bad passes / kappa with E_m >= 1: rejected without a device
    assert lib.amg_setup(ctypes.byref(h), 4, None, None, None, None, 1, 2, None) == amg_mod.AMG_E_ARG
    import numpy as np
    rp = np.array([0, 1, 2], np.int64)
    ci = np.array([0, 1], np.int32)
    v = np.array([1.0, 1.0])
    assert lib.amg_setup(ctypes.byref(h), 2, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, None, 0, 2,
                         None) == amg_mod.AMG_E_ARG
    assert lib.amg_setup(ctypes.byref(h), 2, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, None, 1, 0,
                         None) == amg_mod.AMG_E_ARG
    bad = amg_mod.amg_options_default(kappa=10.0)
    assert lib.amg_setup(ctypes.byref(h), 2, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, None, 1, 2,
                         ctypes.byref(bad)) == amg_mod.AMG_E_ARG
    assert "E_m" in amg_mod.amg_last_error()
    assert lib.amg_free(None) == amg_mod.AMG_OK
    assert lib.amg_solve(None, None, None, 1e-8, 2, None, None) == amg_mod.AMG_E_ARG


def test_product_never_imports_oracle():
    """The product package and the CUDA sources share nothing with oracle/ (DESIGN.md boundary)."""
    pkg = os.path.join(ROOT, "paper_1307_6305_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(//|#).*", "", txt).lower() or f.endswith(".h"), f
                assert "liboracle" not in txt and "import oracle" not in txt and "from oracle" not in txt, f


def test_binding_checks_buffer_lengths(amg_mod):
    """The binding rejects buffers shorter than the CSR / handle sizes before calling into C (a short
    host buffer would otherwise be read or written past its end by the library's copies)."""
    import numpy as np
    import pytest

    rp = np.array([0, 2, 4], np.int64)
    ci = np.array([0, 1, 0, 1], np.int32)
    v = np.array([1.0, -1.0, -1.0, 1.0])
    with pytest.raises(ValueError):
        amg_mod.amg_setup(rp, ci[:3], v, None, 1, 2)
    with pytest.raises(ValueError):
        amg_mod.amg_setup(rp, ci, v[:3], None, 1, 2)
    with pytest.raises(ValueError):
        amg_mod.amg_setup(rp, ci, v, np.zeros(3), 1, 2)
    h = ctypes.c_void_p(1)
    h.n_local = 2
    with pytest.raises(ValueError):
        amg_mod.amg_solve(h, np.zeros(2), np.zeros(1), 1e-8, 2)
    with pytest.raises(ValueError):
        amg_mod.amg_solve(h, np.zeros(3), np.zeros(2), 1e-8, 2)


def test_env_switches_are_documented():
    """Every AMG_* environment switch the library reads appears in DESIGN.md or README.md (DESIGN 7's
    table is the list a reader tunes from; an undocumented switch is an untested code path)."""
    import glob
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    names = set()
    for f in glob.glob(os.path.join(root, "paper_1307_6305_b200", "csrc", "*")):
        names |= set(re.findall(r'getenv\("(AMG_[A-Z0-9_]+)"\)', open(f).read()))
    assert names, "no switches found: the pattern is stale"
    docs = open(os.path.join(root, "DESIGN.md")).read() + open(os.path.join(root, "README.md")).read()
    missing = sorted(n for n in names if n not in docs)
    assert not missing, f"undocumented environment switches: {missing}"

"""The C-ABI library loads and exports every symbol include/efgp.h declares (no GPU needed; no
compute calls).  Also: the binding refuses to run without the library (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "efgp.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(efgp_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("efgp_setup", "efgp_fit", "efgp_predict", "efgp_get_info", "efgp_destroy", "efgp_fit_local",
              "efgp_fit_solve", "efgp_load_weights", "efgp_get_residual_history", "efgp_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2210_10210_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2210_10210_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) <= set(_lib.SIGNATURES)
    assert _lib.load().efgp_abi_version() == 6


def test_library_is_sm100a_only():
    from paper_2210_10210_b200 import _lib
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_missing_library_fails_loudly(tmp_path):
    from paper_2210_10210_b200 import _lib
    saved = _lib._lib
    try:
        _lib._lib = None
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            _lib.load(str(tmp_path / "nope.so"))
    finally:
        _lib._lib = saved


def _struct_fields(name):
    """Field names of `typedef struct { ... } name;` in include/efgp.h, in declaration order."""
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    m = re.search(r"typedef struct \{([^{}]*)\}\s*" + name + r";", src)
    assert m, name
    out = []
    for decl in m.group(1).split(";"):
        decl = decl.strip()
        if not decl:
            continue
        # "double t_spread_ms, t_modes_ms" / "void *stream" / "int64_t nf1, nf2, L"
        first, *rest = [d.strip() for d in decl.split(",")]
        out.append(re.split(r"[\s*]+", first)[-1])
        out.extend(r.lstrip("*").strip() for r in rest)
    return out


@pytest.mark.parametrize("cname,pyname", [("efgp_options", "Options"), ("efgp_info", "Info")])
def test_binding_structs_match_header(cname, pyname):
    # the ctypes mirrors must list the header's fields in the same order (ABI: layout by position)
    from paper_2210_10210_b200 import _lib
    py = [f for f, _ in getattr(_lib, pyname)._fields_]
    assert py == _struct_fields(cname)


@pytest.mark.parametrize("cname,pyname", [("efgp_options", "Options"), ("efgp_info", "Info")])
def test_binding_struct_offsets_match_c(cname, pyname, tmp_path):
    # byte offsets and size of each field as the C compiler lays them out (gcc on the header) equal
    # the ctypes mirror's (catches a type mismatch, not only a name or order mismatch)
    import shutil
    import subprocess
    from paper_2210_10210_b200 import _lib
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    names = _struct_fields(cname)
    src = tmp_path / "off.c"
    body = "".join(f'  printf("%zu\\n", offsetof({cname}, {n}));\n' for n in names)
    src.write_text(f'#include <stdio.h>\n#include <stddef.h>\n#include "{HEADER}"\nint main(void) {{\n{body}'
                   f'  printf("%zu\\n", sizeof({cname}));\n  return 0;\n}}\n')
    exe = tmp_path / "off"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    c_vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    cls = getattr(_lib, pyname)
    py_vals = [getattr(cls, n).offset for n in names] + [ctypes.sizeof(cls)]
    assert py_vals == c_vals


def test_product_path_never_touches_the_oracle():
    # only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may use oracle/;
    # the package and the library sources must not import or mention it as code
    pkg = os.path.join(ROOT, "paper_2210_10210_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f), encoding="utf-8", errors="replace").read()
                assert not re.search(r"^\s*(import oracle|from oracle)", src, flags=re.M), f
    for f in os.listdir(os.path.join(ROOT, "tools")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "tools", f), encoding="utf-8").read()
            assert "import oracle" not in src and "from oracle" not in src and "_util" not in src, f


def test_binding_enums_match_header():
    # the binding's string -> enum maps use the header's values (NEXT-4 preconditioner: G12, G12b)
    import re
    import inspect
    from paper_2210_10210_b200 import efgp as E
    hdr = open(HEADER).read()
    vals = {k: int(v) for k, v in re.findall(r"EFGP_PRECOND_(\w+)\s*=\s*(\d+)", hdr)}
    assert vals == {"NONE": 0, "KRON": 1, "AUTO": 2, "JACOBI": 3}
    src = inspect.getsource(E)
    m = re.search(r"opt\.precond = (\{[^}]*\})", src)
    assert m, "precond map not found in the binding"
    mp = eval(m.group(1))
    for name, v in (("none", "NONE"), ("kron", "KRON"), ("auto", "AUTO"), ("jacobi", "JACOBI")):
        assert mp[name] == vals[v]

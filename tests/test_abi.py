"""C-ABI library checks that need no GPU: the in-tree libmeerkat.so loads and
exports every function include/meerkat.h declares; status strings; create
fails loudly (no CPU fallback) when no device is present; the product package
never imports the oracle."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "meerkat.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(meerkat_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2305_17813_b200 import build, _lib
    build.build()
    return _lib.lib()


def test_header_declares_expected_calls():
    fns = _header_functions()
    from paper_2305_17813_b200 import _lib
    assert fns == sorted(_lib.EXPORTS)
    for must in ("meerkat_create", "meerkat_insert_batch", "meerkat_delete_batch", "meerkat_query_batch",
                 "meerkat_sssp_incremental", "meerkat_sssp_decremental", "meerkat_bfs_incremental",
                 "meerkat_bfs_decremental", "meerkat_destroy"):
        assert must in fns


def test_library_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    syms = set(re.findall(r" T (meerkat_\w+)", out))
    missing = set(_header_functions()) - syms
    assert not missing, missing


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(lib):
    assert lib.meerkat_status_string(0) == b"MEERKAT_OK"
    assert lib.meerkat_status_string(6) == b"MEERKAT_E_STATE"


def test_null_args_rejected(lib):
    from paper_2305_17813_b200 import _lib
    assert lib.meerkat_create(None, None) == _lib.E_INVALID_ARG
    assert lib.meerkat_destroy(None) == _lib.E_INVALID_ARG
    assert lib.meerkat_insert_batch(None, None, None, None, 0, None) == _lib.E_INVALID_ARG
    # seeding mutations: a null graph is rejected before any tree or CUDA state is touched
    assert lib.meerkat_insert_batch_trees(None, None, None, None, 0, None, 0, None) == _lib.E_INVALID_ARG
    assert lib.meerkat_delete_batch_trees(None, None, None, 0, None, 0, None) == _lib.E_INVALID_ARG
    cfg = _lib.Config(vertex_n=0)
    h = ctypes.c_void_p()
    assert lib.meerkat_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.E_INVALID_ARG
    cfg = _lib.Config(vertex_n=10, load_factor=1.5)
    assert lib.meerkat_create(ctypes.byref(cfg), ctypes.byref(h)) == _lib.E_INVALID_ARG


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2305_17813_b200 import Graph, MeerkatError
    with pytest.raises(MeerkatError):
        Graph(16)


def test_product_package_does_not_import_oracle():
    code = ("import sys; import paper_2305_17813_b200, paper_2305_17813_b200.graph; "
            "bad=[m for m in sys.modules if m=='oracle' or m.startswith('oracle.')]; print(bad); assert not bad")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    for f in os.listdir(os.path.join(ROOT, "paper_2305_17813_b200")):
        if f.endswith(".py"):
            assert "import oracle" not in open(os.path.join(ROOT, "paper_2305_17813_b200", f)).read()


def test_ctypes_structs_match_the_header(tmp_path):
    """Every ctypes Structure of the binding has the C layout of include/meerkat.h: a C program built
    from the header prints sizeof / offsetof of each field, compared field by field."""
    import subprocess
    from paper_2305_17813_b200 import _lib
    structs = {"meerkat_config": _lib.Config, "meerkat_stats": _lib.Stats, "meerkat_tree_stats": _lib.TreeStats,
               "meerkat_pagerank_stats": _lib.PageRankStats, "meerkat_latency": _lib.Latency}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "meerkat.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _t in py._fields_:
            lines.append(f'  printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _t in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)

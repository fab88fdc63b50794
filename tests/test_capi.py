"""CPU checks of the boundary: libmeft_cuda.so loads (no GPU needed) and exports exactly the entry points
include/meft_cuda.h declares; the host-side clamp arithmetic mirrors ke_select/topk_select."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "meft_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(meft_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2406_04984_b200 import build

    return build.build()


def test_library_exports_every_declared_symbol(libpath):
    syms = declared_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (meft_[a-z0-9_]+)\b", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # nothing beyond the header leaks out as a C symbol
    assert exported == set(syms), sorted(exported - set(syms))


def test_library_loads_and_binds(libpath):
    from paper_2406_04984_b200 import _lib

    L = _lib.lib()
    assert L.meft_version().decode().startswith("meft-b200")
    assert set(_lib.exported_symbols()) == set(declared_symbols())
    for s in declared_symbols():
        assert hasattr(L, s)


def test_selection_shape_mirrors_reference_clamps(libpath):
    from paper_2406_04984_b200 import meft

    # experts.cpp:56-65: kk_eff = min(kk, N); take = min(K, kk_eff * E); warn when K > visible
    assert meft.selection_shape(4096, 64, 4, 32) == (32, 4, False)
    assert meft.selection_shape(8, 4, 1, 5) == (2, 1, True)
    assert meft.selection_shape(12, 4, 10, 3) == (3, 4, False)
    for bad in [(8, 3, 1, 1), (8, 4, 1, 0), (8, 4, 0, 1), (8, 0, 1, 1)]:
        with pytest.raises(meft.MeftError) as e:
            meft.selection_shape(*bad)
        assert e.value.kind == "invalid_argument"


def test_error_taxonomy_without_gpu(libpath):
    from paper_2406_04984_b200 import _lib

    L = _lib.lib()
    # a null context is rejected with invalid_argument and a readable message, not a crash
    st = L.meft_synchronize(None)
    assert st == 2
    assert "context" in L.meft_last_error(None).decode()


def test_enqueue_only_and_graph_entry_points_reject_null_arguments(libpath):
    """meft_ctx_set_host_sync / meft_graph_* (the enqueue-only step and CUDA graphs) validate before touching CUDA."""
    import ctypes as C

    from paper_2406_04984_b200 import _lib

    L = _lib.lib()
    assert L.meft_ctx_set_host_sync(None, 0) == 2
    assert L.meft_graph_begin(None) == 2
    out = C.c_void_p()
    assert L.meft_graph_end(None, C.byref(out)) == 2
    assert L.meft_graph_launch(None, None) == 2
    assert "context" in L.meft_last_error(None).decode()
    L.meft_graph_destroy(None)  # a no-op, like free(NULL)


def test_header_is_plain_c_and_links(libpath, tmp_path):
    """include/meft_cuda.h is a C header (the FFI boundary): a C11 translation unit compiles against it with
    -pedantic -Werror, links against libmeft_cuda.so and calls into it (argument validation, no GPU needed)."""
    import shutil
    import subprocess

    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    src = tmp_path / "caller.c"
    src.write_text('#include "meft_cuda.h"\n'
                   "int main(void) {\n"
                   "    int peer = 0, overlap = 0;\n"
                   "    meft_graph_destroy((meft_graph*)0);\n"
                   "    if (meft_ctx_sharded_paths((meft_ctx*)0, &peer, &overlap) != MEFT_E_INVALID) return 10;\n"
                   "    return meft_ctx_set_host_sync((meft_ctx*)0, 0) == MEFT_E_INVALID ? 0 : 11;\n"
                   "}\n")
    exe = tmp_path / "caller"
    libdir = os.path.dirname(libpath)
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I",
                        os.path.join(ROOT, "include"), str(src), "-o", str(exe), "-L", libdir, "-lmeft_cuda",
                        "-Wl,-rpath," + libdir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)

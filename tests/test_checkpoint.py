"""MEFT1 checkpoints (memtier.cpp:288-396) through the C ABI's single format implementation (csrc/checkpoint.cu),
pinned byte for byte against files written by the compiled reference (oracle/_ref), and its error taxonomy
(test_memtier.cpp:251-327). Host-only: no GPU needed."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2406_04984_b200 import _lib as L


def _ref_store(train_router, d=16, r=32, n=4, layers=2):
    st = O.RefStore(layers, d, r, n, seed=3, train_router=train_router)
    rng = np.random.default_rng(7)
    for layer in range(layers):  # non-trivial moments and counters: two scatter + Adam rounds
        for _ in range(2):
            s = np.sort(rng.choice(r, 5, replace=False))
            st.scatter_grads(layer, s, rng.standard_normal((d, 5)), rng.standard_normal((5, d)))
            st.sparse_adam(layer, 1e-2)
    return st


def _load(path):
    """meft_ckpt_load into numpy: {(layer, name): array}, header, extra."""
    got = {}

    def sink(user, hp, layer, t, src, n):
        name = L.TENSOR_NAMES[t]
        dt = np.int64 if name.endswith("step") else np.float64
        got[(layer, name)] = np.ctypeslib.as_array(C.cast(src, C.POINTER(C.c_int64 if dt is np.int64 else C.c_double)),
                                                   shape=(n,)).astype(dt).copy()
        return 0

    cb = L.CKPT_SINK(sink)
    hdr, extra = L.CkptHeader(), C.create_string_buffer(4096)
    st = L.lib().meft_ckpt_load(str(path).encode(), C.byref(hdr), extra, len(extra), cb, None)
    return st, got, hdr, extra.value.decode()


def _save(path, got, hdr, extra):
    def source(user, layer, t, dst, n):
        a = got[(layer, L.TENSOR_NAMES[t])]
        C.memmove(dst, a.ctypes.data, n * 8)
        return 0

    cb = L.CKPT_SOURCE(source)
    return L.lib().meft_ckpt_save(str(path).encode(), C.byref(hdr), extra.encode(), cb, None)


@pytest.mark.parametrize("train_router", [False, True])
def test_format_round_trip_is_byte_identical_to_reference(tmp_path, train_router):
    ref = _ref_store(train_router)
    a, b = tmp_path / "ref.meft", tmp_path / "ours.meft"
    ref.save(a, extra='{"run": "x", "k": [1, 2.5, true, null]}', step=42)
    st, got, hdr, extra = _load(a)
    assert st == 0, L.lib().meft_last_error(None)
    assert (hdr.layers, hdr.dim, hdr.pairs, hdr.experts, hdr.step, hdr.train_router) == (2, 16, 32, 4, 42,
                                                                                          int(train_router))
    np.testing.assert_array_equal(got[(1, "m_a")].reshape(16, 32), ref.get(1, "m_a"))
    np.testing.assert_array_equal(got[(0, "pair_step")], ref.pair_step(0))
    assert _save(b, got, hdr, extra) == 0
    assert a.read_bytes() == b.read_bytes()


REAL_EXTRAS = [
    '{"lr": 0.001, "eps": 1e-08, "b1": 0.9, "b2": 0.999, "big": 1e+20, "e15": 1e15, "e16": 12345678901234567.0}',
    '{"x": [0.1, 0.2, 0.30000000000000004, -0.0, 0.0, 100.0, 1.5, 123456.789, 5e-324, 1.7976931348623157e308]}',
    '{"small": [0.0001, 0.00001, 2.5e-4, 1e-3], "name": "caf\\u00e9 \\ud83d\\ude00"}',
]


@pytest.mark.parametrize("extra", REAL_EXTRAS)
def test_header_reals_and_unicode_are_byte_identical_to_reference(tmp_path, extra):
    """The header's `extra` (e.g. the run config echo with lr, eps) is re-serialised by nlohmann in the reference:
    reals in their shortest round-trip form, \\u surrogate pairs decoded to one UTF-8 code point."""
    ref = _ref_store(False, layers=1)
    a, b = tmp_path / "ref.meft", tmp_path / "ours.meft"
    ref.save(a, extra=extra, step=3)
    st, got, hdr, ex = _load(a)
    assert st == 0, L.lib().meft_last_error(None)
    assert _save(b, got, hdr, ex) == 0
    assert a.read_bytes().split(b"\n", 1)[0] == b.read_bytes().split(b"\n", 1)[0]
    assert a.read_bytes() == b.read_bytes()


def _corrupt(tmp_path, name, transform):
    ref = _ref_store(False)
    p = tmp_path / name
    ref.save(p)
    p.write_bytes(transform(p.read_bytes()))
    return p


@pytest.mark.parametrize("case,code", [
    ("bad_magic", 9), ("version", 9), ("missing_field", 9), ("corrupt_header", 9), ("empty", 9),
    ("truncated", 11), ("trailing", 10), ("zero_shape", 10),
])
def test_error_taxonomy(tmp_path, case, code):
    def edit(b):
        head, body = b.split(b"\n", 1)
        if case == "bad_magic":
            return head.replace(b"MEFT1", b"MEFT2") + b"\n" + body
        if case == "version":
            return head.replace(b'"version":1', b'"version":2') + b"\n" + body
        if case == "missing_field":
            return head.replace(b'"pairs":32,', b"") + b"\n" + body
        if case == "corrupt_header":
            return head[:-5] + b"\n" + body
        if case == "empty":
            return b""
        if case == "truncated":
            return b[:-9]
        if case == "trailing":
            return b + b"x"
        if case == "zero_shape":
            return head.replace(b'"dim":16', b'"dim":0') + b"\n" + body
        raise AssertionError(case)

    p = _corrupt(tmp_path, case, edit)
    st, _, _, _ = _load(p)
    assert st == code, (st, L.lib().meft_last_error(None))


def test_extra_must_be_json_and_missing_file_is_io(tmp_path):
    hdr = L.CkptHeader(1, 4, 8, 2, 0, 0)
    cb = L.CKPT_SOURCE(lambda *a: 0)
    assert L.lib().meft_ckpt_save(str(tmp_path / "x").encode(), C.byref(hdr), b"{not json", cb, None) == 2
    st, _, _, _ = _load(tmp_path / "does_not_exist")
    assert st == 12

"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports
every symbol include/a2ats.h declares, and rejects bad arguments before any
CUDA call (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "a2ats.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2502_12665_b200 import binding, build
    build.build()
    return binding.load()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(a2ats_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("a2ats_build_codes", "a2ats_decode_step", "a2ats_qavq_prepare", "a2ats_decode_workspace_bytes",
              "a2ats_build_codes_workspace_bytes", "a2ats_status_string", "a2ats_default_params"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (a2ats_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_sm100a_code_present(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version(lib):
    from paper_2502_12665_b200 import binding as b
    assert lib.a2ats_abi_version() == b.ABI_VERSION == 10
    for s in (b.A2ATS_OK, b.A2ATS_EINVAL, b.A2ATS_EUNSUPPORTED, b.A2ATS_EWORKSPACE, b.A2ATS_ECUDA, b.A2ATS_ENCCL):
        assert b.status_string(s).startswith("A2ATS")


def test_default_params_are_the_papers(lib, golden):
    from paper_2502_12665_b200 import binding as b
    g = golden("paper_constants.json")
    p = b.a2ats_params()
    lib.a2ats_default_params(ctypes.byref(p))
    assert (p.window, p.bridge, p.n_sink) == (g["window"], g["bridge"], g["n_sink"])
    assert p.rope_theta == 1e4 and p.group_reduce == b.A2ATS_GROUP_MAX


def _call_decode(lib, shape, params, n_ctx, ws_bytes=1 << 40, null_q=False, ws=True):
    from paper_2502_12665_b200 import binding as b
    fake = 1 << 20      # 16-byte aligned, never dereferenced: validation fails first
    return lib.a2ats_decode_step(ctypes.byref(shape), ctypes.byref(params), n_ctx, None if null_q else fake, fake, fake,
                                 fake, fake, None, fake, None, None, fake if ws else None, ws_bytes, None)


def test_validation_without_gpu(lib):
    from paper_2502_12665_b200 import binding as b
    p = b.Params(topk=100).c()
    good = b.make_shape(2, 32, 8, 128, 4096, 32768)
    assert lib.a2ats_decode_workspace_bytes(ctypes.byref(good), ctypes.byref(p)) > 0
    assert _call_decode(lib, b.make_shape(2, 32, 8, 64, 4096, 32768), p, 100) == b.A2ATS_EUNSUPPORTED
    assert _call_decode(lib, b.make_shape(2, 32, 8, 127, 4096, 32768), p, 100) == b.A2ATS_EINVAL
    assert _call_decode(lib, b.make_shape(2, 30, 8, 128, 4096, 32768), p, 100) == b.A2ATS_EINVAL
    assert _call_decode(lib, b.make_shape(2, 24, 8, 128, 4096, 32768), p, 100) == b.A2ATS_EUNSUPPORTED  # G = 3
    assert _call_decode(lib, b.make_shape(2, 32, 8, 128, 4096, 32767), p, 100) == b.A2ATS_EINVAL       # n_max % 8
    assert _call_decode(lib, good, p, 0) == b.A2ATS_EINVAL
    assert _call_decode(lib, good, p, 32769) == b.A2ATS_EINVAL
    assert _call_decode(lib, good, p, 100, null_q=True) == b.A2ATS_EINVAL
    assert _call_decode(lib, good, p, 100, ws=False) == b.A2ATS_EWORKSPACE
    assert _call_decode(lib, good, p, 100, ws_bytes=16) == b.A2ATS_EWORKSPACE
    bad = b.Params(topk=-1).c()
    assert _call_decode(lib, good, bad, 100) == b.A2ATS_EINVAL
    fake = 1 << 20
    assert lib.a2ats_qavq_prepare(ctypes.byref(good), fake, None, fake, None, None) == b.A2ATS_EINVAL  # no chat
    assert lib.a2ats_build_codes(ctypes.byref(good), fake, 10, 5, fake, fake, fake, None, fake, 1 << 40,
                                 None) == b.A2ATS_EINVAL
    assert lib.a2ats_build_codes(ctypes.byref(good), fake, 0, 32769, fake, fake, fake, None, fake, 1 << 40,
                                 None) == b.A2ATS_EINVAL
    assert lib.a2ats_build_codes(ctypes.byref(good), fake, 0, 10, fake, fake, fake, None, fake, 8,
                                 None) == b.A2ATS_EWORKSPACE
    assert lib.a2ats_build_codes(ctypes.byref(good), fake, 5, 5, fake, fake, fake, None, fake, 1 << 40,
                                 None) == b.A2ATS_OK     # empty range: nothing to do


def test_workspace_size_grows_with_budget(lib):
    from paper_2502_12665_b200 import binding as b
    s = b.make_shape(16, 32, 8, 128, 4096, 32768)
    small = b.a2ats_decode_workspace_bytes(s, b.Params(topk=100))
    big = b.a2ats_decode_workspace_bytes(s, b.Params(topk=2000))
    assert big > small > 0
    assert b.a2ats_build_codes_workspace_bytes(s) > 0


def test_round2_abi_fields_without_gpu(lib):
    """ABI 9 fields validated on the host: code width (uint8 only for L <= 256), hist_lag (deferred
    a0, at most the window), per-query-head mode (its own workspace layout), padded posting rows."""
    from paper_2502_12665_b200 import binding as b
    p = b.Params(topk=100)
    assert b.a2ats_decode_workspace_bytes(b.make_shape(2, 8, 2, 128, 256, 4096, code_bytes=1), p) > 0
    assert b.a2ats_decode_workspace_bytes(b.make_shape(2, 8, 2, 128, 300, 4096, code_bytes=1), p) == 0
    assert b.a2ats_decode_workspace_bytes(b.make_shape(2, 8, 2, 128, 256, 4096, code_bytes=3), p) == 0
    s = b.make_shape(2, 8, 2, 128, 1000, 4096)
    assert b.a2ats_decode_workspace_bytes(s, b.Params(topk=100, hist_lag=64)) > 0
    assert b.a2ats_decode_workspace_bytes(s, b.Params(topk=100, hist_lag=65)) == 0
    assert b.a2ats_decode_workspace_bytes(s, b.Params(topk=100, hist_lag=-1)) == 0
    gqa = b.a2ats_decode_workspace_bytes(s, b.Params(topk=100))
    per_head = b.a2ats_decode_workspace_bytes(s, b.Params(topk=100, group_reduce=b.A2ATS_GROUP_PER_HEAD))
    assert per_head > 0 and gqa > 0 and per_head != gqa  # (the sub-step's own layout + q / out / sel buffers)
    assert b.a2ats_decode_workspace_bytes(s, b.Params(topk=100, group_reduce=3)) == 0
    # posting index: offsets [P, (L + 4) & ~3] int32, then (256-B aligned) tokens [P, n_max] int32
    P, LP = 4, (1000 + 4) // 4 * 4
    tok = (P * LP * 4 + 255) // 256 * 256
    assert b.a2ats_postings_bytes(s) == (tok + P * 4096 * 4 + 255) // 256 * 256

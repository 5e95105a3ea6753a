"""CPU checks of the C-ABI library: it loads, exports every symbol include/shiftadd.h declares,
and its host-side logic (sizes, validation) behaves -- no compute calls (no GPU here)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shiftadd.h")
LIBPATH = os.path.join(ROOT, "paper_2406_05981_b200", "libshiftadd.so")


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(LIBPATH):
        import __graft_entry__
        __graft_entry__.build()
    import paper_2406_05981_b200 as sa
    return sa.lib()


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(shiftadd_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_section8b_entry_points():
    names = _declared()
    for must in ("shiftadd_pack", "shiftadd_lut_gemv", "shiftadd_lut_gemm", "shiftadd_workspace_bytes",
                 "shiftadd_abi_version", "shiftadd_status_string", "shiftadd_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    out = subprocess.run(["nm", "-D", "--defined-only", LIBPATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (shiftadd_\w+)", out))
    for name in _declared():
        assert name in exported, name
        assert hasattr(L, name)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIBPATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_abi_version_and_status_strings(L):
    assert L.shiftadd_abi_version() == 1
    assert L.shiftadd_status_string(0) == b"ok"
    assert L.shiftadd_status_string(2) == b"invalid argument"
    assert L.shiftadd_status_string(6) == b"unsupported"
    assert L.shiftadd_status_string(7) == b"cuda error"


@pytest.mark.parametrize("q,N,K,g", [(3, 768, 768, 128), (2, 4096, 4096, 128), (3, 11008, 4096, 128),
                                     (1, 33, 512, 256), (4, 17, 256, 256)])
def test_packed_bytes_match_oracle_accounting(L, q, N, K, g):
    e = ctypes.c_size_t()
    assert L.shiftadd_packed_bytes(0, q, N, K, g, ctypes.byref(e)) == oracle.packed_bytes(q, N, K, g)[0]
    assert e.value == oracle.packed_bytes(q, N, K, g)[1]
    p = L.shiftadd_packed_bytes(1, q, N, K, g, ctypes.byref(e))
    assert (p, e.value) == oracle.tiled_sizes(q, N, K)


def test_packed_bytes_rejects_bad_shapes(L):
    e = ctypes.c_size_t()
    assert L.shiftadd_packed_bytes(0, 3, 768, 100, 128, ctypes.byref(e)) == 0   # K % 8
    assert L.shiftadd_packed_bytes(1, 3, 768, 768, 64, ctypes.byref(e)) == 0    # tiled needs 128 | g
    assert L.shiftadd_packed_bytes(1, 3, 768, 640, 128, ctypes.byref(e)) == 0   # tiled needs 256 | K
    assert L.shiftadd_packed_bytes(0, 9, 768, 768, 128, ctypes.byref(e)) == 0   # q <= 8
    assert b"q=9" in L.shiftadd_last_error()


def test_workspace_bytes(L):
    # tiled M=1 (streaming kernel): counter region + gather counter + epoch word + {epoch,
    # fp32} partials [RG][S][16]; S == 1 needs none.  Every kernel's partials start after the
    # epoch word (kPartOff = 256 KB + 512), so none overwrites another's carried-over state.
    S, RG = 4096 // 256, 4096 // 16
    C = 65536 * 4  # per-row-group counters
    assert L.shiftadd_workspace_bytes(1, 1, 4096, 4096, 3, 128) == C + 256 + 256 + S * RG * 16 * 8
    assert L.shiftadd_workspace_bytes(1, 1, 4096, 256, 3, 128) == 0
    assert L.shiftadd_workspace_bytes(1, 8, 4096, 4096, 3, 128) == C + 512 + 8 * S * RG * 16 * 8
    # M = 16: the larger of the streaming kernel (two row chunks of 8 reuse one region) and the
    # small-batch split-K kernel (fp32 partials for all 16 rows)
    assert L.shiftadd_workspace_bytes(1, 16, 4096, 4096, 3, 128) == max(C + 512 + 8 * S * RG * 16 * 8,
                                                                        C + 512 + 16 * S * RG * 16 * 4)
    assert L.shiftadd_workspace_bytes(0, 1, 4096, 4096, 3, 128) == 0
    assert L.shiftadd_workspace_bytes(1, 17, 4096, 4096, 3, 128) == 0


def _buf(n, align=256):
    raw = ctypes.create_string_buffer(n + align)
    addr = (ctypes.addressof(raw) + align - 1) // align * align
    return raw, ctypes.c_void_p(addr)


def test_gemm_validation_happens_before_any_launch(L):
    _r1, p = _buf(1 << 16)
    _r2, p_odd = _buf(1 << 16)
    odd = ctypes.c_void_p(p_odd.value + 2)
    # null pointers
    assert L.shiftadd_lut_gemm(None, 768, p, p, 1, 1, 768, 768, 3, 128, p, 768, None, 0, 0, None) == 2
    # q out of range, M too large, ld too small, bad layout, unknown flags, misaligned x
    assert L.shiftadd_lut_gemm(p, 768, p, p, 1, 1, 768, 768, 5, 128, p, 768, None, 0, 0, None) == 2
    assert L.shiftadd_lut_gemm(p, 768, p, p, 1, 17, 768, 768, 3, 128, p, 768, None, 0, 0, None) == 6
    assert L.shiftadd_lut_gemm(p, 700, p, p, 1, 1, 768, 768, 3, 128, p, 768, None, 0, 0, None) == 2
    assert L.shiftadd_lut_gemm(p, 768, p, p, 7, 1, 768, 768, 3, 128, p, 768, None, 0, 0, None) == 2
    assert L.shiftadd_lut_gemm(p, 768, p, p, 1, 1, 768, 768, 3, 128, p, 768, None, 0, 8, None) == 2
    assert L.shiftadd_lut_gemm(odd, 768, p, p, 1, 1, 768, 768, 3, 128, p, 768, None, 0, 0, None) == 2
    # missing workspace for a split-K shape
    assert L.shiftadd_lut_gemm(p, 4096, p, p, 1, 1, 4096, 4096, 3, 128, p, 4096, None, 0, 0, None) == 2
    assert b"workspace" in L.shiftadd_last_error()
    # pack: bad sign alignment / null
    assert L.shiftadd_pack(None, p, 3, 16, 256, 128, 1, p, p, None, None) == 2
    assert L.shiftadd_pack(odd, p, 3, 16, 256, 128, 1, p, p, None, None) == 2


def test_valid_call_without_a_gpu_reports_cuda_error(L):
    _r, p = _buf(1 << 20)
    st = L.shiftadd_lut_gemm(p, 768, p, p, 0, 1, 768, 768, 3, 128, p, 768, None, 0, 0, None)
    assert st == 7 and len(L.shiftadd_last_error()) > 0


def test_python_binding_fails_loudly_without_gpu_tensors():
    import torch
    import paper_2406_05981_b200 as sa
    with pytest.raises(ValueError):
        sa.pack(torch.ones((1, 16, 256), dtype=torch.int8), torch.ones((1, 16, 2)), 128)


def test_colwise_validation_happens_before_any_launch(L):
    _r1, p = _buf(1 << 16)
    # null pointers, bad q, canonical layout (the column-wise GEMV is tiled-only)
    assert L.shiftadd_pack_colwise(None, p, 3, 16, 256, 1, p, p, None, None) == 2
    assert L.shiftadd_pack_colwise(p, p, 9, 16, 256, 1, p, p, None, None) == 2
    assert L.shiftadd_pack_colwise(p, p, 3, 16, 250, 1, p, p, None, None) == 2
    assert L.shiftadd_lut_gemv_colwise(None, p, p, 1, 16, 256, 3, p, 0, None) == 2
    assert L.shiftadd_lut_gemv_colwise(p, p, p, 1, 16, 256, 5, p, 0, None) == 2
    assert L.shiftadd_lut_gemv_colwise(p, p, p, 0, 16, 256, 3, p, 0, None) == 6
    assert L.shiftadd_lut_gemv_colwise(p, p, p, 1, 16, 256, 3, p, 8, None) == 2
    assert b"flags" in L.shiftadd_last_error()


def test_apot2_validation_happens_before_any_launch(L):
    _r1, p = _buf(1 << 16)
    assert L.shiftadd_pack_apot2(p, p, 3, 16, 256, 128, 1, p, p, None, None, None) == 2
    assert L.shiftadd_lut_gemm_apot2(p, 512, p, p, None, 1, 1, 64, 512, 3, 128, p, 64, 0, None) == 2
    assert L.shiftadd_lut_gemm_apot2(p, 512, p, p, p, 1, 2, 64, 512, 3, 128, p, 64, 0, None) == 6
    assert L.shiftadd_lut_gemm_apot2(p, 512, p, p, p, 1, 1, 64, 512, 3, 128, p, 64, 8, None) == 2   # unknown flag
    # the workspace form: K > 4096 tiled needs the workspace (streaming kernel), validated on the host
    assert L.shiftadd_workspace_bytes_apot2(64, 8192) > 0
    assert L.shiftadd_lut_gemm_apot2_ws(p, 8192, p, p, p, 1, 1, 64, 8192, 3, 128, p, 64, p, 16, 8, None) == 2
    assert L.shiftadd_lut_gemm_apot2_ws(p, 8192, p, p, p, 1, 2, 64, 8192, 3, 128, p, 64, p, 1 << 16, 0, None) == 6


def test_quantize_validation_happens_before_any_launch(L):
    _r1, p = _buf(1 << 16)
    assert L.shiftadd_bcq_quantize(None, 4, 256, 2, 128, 3, 0, p, p, None) == 2
    assert L.shiftadd_bcq_quantize(p, 4, 256, 5, 128, 3, 0, p, p, None) == 2
    assert L.shiftadd_bcq_quantize(p, 4, 256, 2, 100, 3, 0, p, p, None) == 2
    assert L.shiftadd_bcq_quantize(p, 4, 256, 2, 128, -1, 0, p, p, None) == 2
    assert L.shiftadd_bcq_quantize(p, 4, 256, 2, 128, 3, 4, p, p, None) == 2
    assert L.shiftadd_bcq_quantize(p, 4, 256, 2, 128, 3, 1, p, p, None) == 7   # valid: no GPU here


def test_gather_validation_happens_before_any_launch(L):
    _r1, p = _buf(1 << 20)
    args = (p, p, p, 1, 4096, 4096, 3, 128)
    assert L.shiftadd_lut_gemv_gather(*args, None, p, 2, 0, p, p, 1 << 19, 0, None) == 2
    assert L.shiftadd_lut_gemv_gather(*args, p, p, 2, 0, None, p, 1 << 19, 0, None) == 2  # no epoch counter
    assert L.shiftadd_lut_gemv_gather(*args, p, p, 1, 0, p, p, 1 << 19, 0, None) == 2     # P < 2
    assert L.shiftadd_lut_gemv_gather(*args, p, p, 2, 2, p, p, 1 << 19, 0, None) == 2     # rank >= P
    assert L.shiftadd_lut_gemv_gather(*args, p, p, 2, 0, p, p, 1024, 0, None) == 2        # workspace
    assert L.shiftadd_lut_gemv_gather(p, p, p, 0, 4096, 4096, 3, 128, p, p, 2, 0, p, p, 1 << 19, 0, None) == 6
    assert L.shiftadd_gather_wait(None, 2, p, None) == 2


def test_copy_validation_happens_before_any_launch(L):
    _r1, p = _buf(1 << 16)
    q = ctypes.c_void_p(p.value + 8)
    assert L.shiftadd_copy(None, p, 256, 0, None) == 2          # null pointer
    assert L.shiftadd_copy(p, p, 100, 0, None) == 2             # not a multiple of 16
    assert L.shiftadd_copy(q, p, 256, 0, None) == 2             # misaligned
    assert L.shiftadd_copy(p, p, 256, 8, None) == 2             # unknown flag
    assert L.shiftadd_copy(p, p, 256, 1 | 4, None) == 7         # valid: no GPU here


def test_program_encode_and_validation_happen_on_the_host(L):
    """Decode program (kernel 9): encoding is host-only (no GPU needed), sizes follow the call
    list, and every malformed call is rejected before any launch."""
    import paper_2406_05981_b200 as sa
    calls = (sa._Call * 2)()
    fake = 1 << 20   # never dereferenced on the host
    for j, (K, segs) in enumerate([(4096, [(4096, 2), (4096, 3), (4096, 2)]), (11008, [(4096, 2)])]):
        c = calls[j]
        c.x, c.K, c.g, c.nseg, c.flags = fake, K, 128, len(segs), sa.CALL_WAIT if j else 0
        for i, (N, q) in enumerate(segs):
            c.seg[i] = sa._Segment(fake, fake, N, q, fake)
    nb = L.shiftadd_program_bytes(2)
    assert nb == 2 * L.shiftadd_program_bytes(1) - 64 and L.shiftadd_program_bytes(0) == 0
    buf = (ctypes.c_uint8 * nb)()
    assert L.shiftadd_program_encode(calls, 2, ctypes.addressof(buf), nb) == 0
    assert bytes(buf[:8]) == b"SPRGS201"   # header magic
    # workspace: 256 + two regions of max S x RGtot x 16 x 8 B (the q/k/v call: 16 x 768)
    ws = L.shiftadd_workspace_bytes_program(calls, 2)
    region = max(16 * 768, 43 * 256) * 16 * 8
    assert ws == 256 + 2 * ((region + 255) // 256 * 256)
    assert L.shiftadd_program_encode(calls, 2, ctypes.addressof(buf), nb - 1) == 2   # buffer too small
    calls[1].flags = 8
    assert L.shiftadd_program_encode(calls, 2, ctypes.addressof(buf), nb) == 2       # unknown flag
    calls[1].flags = 0
    calls[1].K = 11000
    assert L.shiftadd_program_encode(calls, 2, ctypes.addressof(buf), nb) == 2       # K % 256
    calls[1].K = 11008
    calls[0].seg[1].q = 5
    assert L.shiftadd_program_encode(calls, 2, ctypes.addressof(buf), nb) == 2       # q outside 1..4
    calls[0].seg[1].q = 3
    calls[0].nseg = 5
    assert L.shiftadd_program_encode(calls, 2, ctypes.addressof(buf), nb) == 2
    calls[0].nseg = 3
    calls[0].x = fake + 2
    assert L.shiftadd_program_encode(calls, 2, ctypes.addressof(buf), nb) == 2       # x alignment
    calls[0].x = fake
    assert L.shiftadd_program_encode(calls, 0, ctypes.addressof(buf), nb) == 2
    # a valid program on a machine without a GPU: the launch reports a CUDA error, no crash
    assert L.shiftadd_lut_gemv_program(calls, 2, fake, nb, fake, ws, 0, None) == 7


def test_round2_entry_points_validate_before_any_launch(L):
    """Column-wise with a workspace (any K, M <= 16), fused gather for M <= 8, fused segments:
    malformed calls are rejected on the host; well-formed ones reach the device check."""
    _r1, p = _buf(1 << 20)
    ws = 1 << 19
    assert L.shiftadd_workspace_bytes_colwise(4096, 8192) == 256 * 1024 + 256 + 256 + 2 * 32 * 256 * 16 * 8
    assert L.shiftadd_workspace_bytes_colwise(4096, 8000) == 0
    # column-wise M = 1 (workspace form) and M <= 16
    assert L.shiftadd_lut_gemv_colwise_ws(None, p, p, 1, 64, 8192, 3, p, p, ws, 0, None) == 2
    assert L.shiftadd_lut_gemv_colwise_ws(p, p, p, 1, 64, 8192, 3, p, p, ws, 16, None) == 2      # unknown flag
    assert L.shiftadd_lut_gemv_colwise_ws(p, p, p, 0, 64, 8192, 3, p, p, ws, 0, None) == 6       # canonical
    assert L.shiftadd_lut_gemm_colwise(p, 8192, p, p, 1, 17, 64, 8192, 3, p, 64, p, ws, 0, None) == 6   # M > 16
    assert L.shiftadd_lut_gemm_colwise(p, 8000, p, p, 1, 4, 64, 8192, 3, p, 64, p, ws, 0, None) == 2    # ldx < K
    assert L.shiftadd_lut_gemm_colwise(p, 8192, p, p, 1, 4, 64, 8192, 3, p, 32, p, ws, 0, None) == 2    # ldy < N
    assert L.shiftadd_lut_gemm_colwise(p, 8192, p, p, 1, 4, 64, 8192, 3, p, 64, p, ws, 0, None) == 7    # valid
    # fused gather, M <= 8
    g = (p, p, 2, 0, p, p, ws, 0, None)
    assert L.shiftadd_lut_gemm_gather(p, 4096, p, p, 1, 9, 64, 4096, 3, 128, *g) == 6          # M > 8
    assert L.shiftadd_lut_gemm_gather(p, 4000, p, p, 1, 3, 64, 4096, 3, 128, *g) == 2          # ldx < K
    assert L.shiftadd_lut_gemm_gather(p, 4096, p, p, 1, 3, 64, 4096, 3, 128, *g) == 7          # valid
    # fused segments: unknown flag, too many segments
    import paper_2406_05981_b200 as sa
    segs = (sa._Segment * 5)()
    assert L.shiftadd_lut_gemv_fused(p, 4096, 128, 1, 5, segs, p, ws, 0, None) == 2
    for i in range(2):
        segs[i] = sa._Segment(p.value, p.value, 64, 2, p.value)
    assert L.shiftadd_lut_gemv_fused(p, 4096, 128, 1, 2, segs, p, ws, 8, None) == 2              # unknown flag
    assert L.shiftadd_lut_gemv_fused(p, 4096, 128, 1, 2, segs, p, ws, 2, None) == 7              # SPLITK: valid

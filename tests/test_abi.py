"""C-ABI surface checks that need no GPU: the library loads, exports every
symbol include/zstripe_b200.h declares, and rejects bad arguments with the
documented zs_status codes before touching a device."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "zstripe_b200.h"

from paper_2605_17633_b200 import _lib  # noqa: E402


def header_symbols():
    return sorted(set(re.findall(r"^ZS_API\s+(?:const\s+char\s*\*|int|size_t|unsigned\s+long\s+long)\s+(zs_\w+)\(", HEADER.read_text(), re.M)))


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        pytest.fail(f"{_lib.LIB_PATH} not built (run __graft_entry__.build())")
    return _lib.load()


def test_header_declares_the_hot_path():
    syms = header_symbols()
    for s in ("zs_sobel_saliency", "zs_rank_order", "zs_permute_rows_f32", "zs_layout_maps", "zs_prefix_keep_rows",
              "zs_layernorm_rows", "zs_gemm_bf16", "zs_stripe_attn_fwd", "zs_rc_mlp_fwd", "zs_status_string"):
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert sorted(_lib.exported_symbols()) == header_symbols()


def test_binding_arity_matches_header(lib):
    text = HEADER.read_text()
    for name, args in _lib.SIGNATURES.items():
        m = re.search(rf"ZS_API\s+(?:int|size_t|unsigned\s+long\s+long)\s+{name}\(([^;]*)\);", text, re.S)
        assert m, name
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), (name, len(params), len(args))


def test_status_strings(lib):
    assert _lib.status_string(0) == "ok"
    for code in (-1, -2, -3, -4, -5, -6, -7):
        assert "unknown" not in _lib.status_string(code)
    assert "unknown" in _lib.status_string(-99)
    assert lib.zs_abi_version() == _lib.ABI_VERSION == 200


def test_workspace_queries(lib):
    # window attention: fp16 operand rows [heads*S + S, 32]; global: [heads*S, 128]; per-unit tables scale by units
    assert lib.zs_stripe_attn_ws_bytes(25, 16, 196, 196, 80, 0) == (16 * 196 + 196) * 32 * 2
    assert lib.zs_stripe_attn_ws_bytes(25, 16, 196, 196, 80, 1) == -(-(25 * 16 * 196 + 196) * 64 // 256) * 256
    assert lib.zs_stripe_attn_ws_bytes(64, 16, 4096, 4096, 80, 0) == 16 * 4096 * 128 * 2
    assert lib.zs_stripe_attn_ws_bytes(64, 16, 4096, 4096, 32, 0) == 0  # unsupported head dim
    assert lib.zs_relpos_ws_bytes(4, 16, 4096, 80, 64) >= lib.zs_stripe_attn_ws_bytes(4, 16, 4096, 4096, 80, 1)
    assert isinstance(lib.zs_launch_counter(), int)  # per-thread counter, readable without a device


def test_missing_workspace_is_an_error_not_an_allocation(lib):
    # a window-attention call that passes the shape checks but no workspace -> ZS_ERR_WORKSPACE
    # (the library never allocates); checked before any device work
    fake = ctypes.c_void_p(0x1000)
    args = [fake, fake, fake, 64 * 16, 64 * 16, 64 * 16, 0, 0, 1, 16, 196, 196, 64, fake, fake, 14, fake, fake, 32, 32,
            2, 0.125, fake, 64 * 16, 0, None, 0, None]
    rc = lib.zs_stripe_attn_fwd(*args)
    assert rc == -7, _lib.status_string(rc)


def test_argument_errors_without_device(lib):
    fake = ctypes.c_void_p(0x1000)
    # GEMM: null operand -> ZS_ERR_ARG; K % 64 != 0 -> ZS_ERR_SHAPE
    assert lib.zs_gemm_bf16(0, None, 64, fake, 64, 8, 64, 64, None, fake, 64, None, 0, None, None, 0, None,
                            None) == -1
    assert lib.zs_gemm_bf16(0, fake, 100, fake, 100, 8, 64, 100, None, fake, 64, None, 0, None, None, 0, None,
                            None) == -2
    # attention: head dim 32 unsupported -> ZS_ERR_SHAPE; bias grid w*w != Sk -> ZS_ERR_SHAPE
    args = [fake, fake, fake, 64, 64, 64, 0, 0, 1, 1, 16, 16, 32, fake, fake, 4, fake, fake, 8, 8, 1, 0.1, fake, 64,
            0, fake, 1 << 20, None]
    assert lib.zs_stripe_attn_fwd(*args) == -2
    args[12] = 64
    args[15] = 3
    assert lib.zs_stripe_attn_fwd(*args) == -2
    # rank order: g must divide N
    assert lib.zs_rank_order(fake, 0, 1, 10, 0, 2, 4, 0, fake, fake, None, None) == -2
    # permute: C not a multiple of 4
    assert lib.zs_permute_rows_f32(fake, fake, fake, 5, 6, None) == -2
    # empty work is a no-op success
    assert lib.zs_permute_rows_f32(fake, fake, fake, 0, 6, None) == 0

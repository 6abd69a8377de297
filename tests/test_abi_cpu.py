"""CPU-side checks of the C-ABI boundary: the library builds/loads and exports every
symbol include/puzzlemoe.h declares; host-only calls work without a device; argument
errors are rejected synchronously before any launch; compute calls fail loudly (no CPU
fallback) when no device exists."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "puzzlemoe.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2511_04805_b200 import build
    build.build()
    import paper_2511_04805_b200 as pz
    return pz.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(puzzle_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ("puzzle_merge_pack", "puzzle_unpack", "puzzle_moe_forward"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    import paper_2511_04805_b200 as pz
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert sorted(pz.EXPORTED_SYMBOLS) == declared_functions()


def test_host_only_calls(lib):
    assert lib.puzzle_abi_version() >> 16 == 1
    assert lib.puzzle_status_string(0) == b"PUZZLE_OK"
    assert lib.puzzle_status_string(4) == b"PUZZLE_ERR_WORKSPACE"
    import paper_2511_04805_b200 as pz
    desc = pz.MoELayerDesc(8, 4, 4096, 14336, 4096, 4096, 4096)  # fake aligned addresses, never dereferenced
    ws = lib.puzzle_moe_workspace_size(ctypes.byref(desc), 64, 2)
    # must at least hold h (bf16) and y (f32) for the 128 assignments
    assert ws >= 128 * 14336 * 2 + 128 * 4096 * 4
    bad = pz.MoELayerDesc(8, 4, 4000, 14336, 4096, 4096, 4096)  # d_model % 64 != 0
    assert lib.puzzle_moe_workspace_size(ctypes.byref(bad), 64, 2) == 0


def test_argument_errors_are_synchronous(lib):
    assert lib.puzzle_unpack(None, 2, 10, None, None) == 1            # pos not in {0,1}
    assert b"pos" in lib.puzzle_last_error()
    assert lib.puzzle_unpack(None, 0, 0, None, None) == 0             # n == 0: no-op
    assert lib.puzzle_merge_pack(None, None, None, None, None, -1, None, None, None) == 1
    assert lib.puzzle_merge_experts_pack(None, None, None, None, 1, 1, 8, ctypes.c_float(1.5), None, None, None) == 1
    import paper_2511_04805_b200 as pz
    desc = pz.MoELayerDesc(9, 4, 4096, 14336, 4096, 4096, 4096)     # E > 2P
    assert lib.puzzle_moe_forward(ctypes.byref(desc), None, None, 1, 2, 1, None, None, None, 0, None) == 1
    # E < 2P (the 25% ratio: merged pairs + dense slots, R20) is a valid layer: sizes only
    desc = pz.MoELayerDesc(8, 6, 4096, 14336, 4096, 4096, 4096, 4096)
    assert lib.puzzle_moe_workspace_size(ctypes.byref(desc), 64, 2) > 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_compute_without_device_fails_loudly(lib):
    buf = (ctypes.c_uint16 * 8)()
    out = (ctypes.c_uint16 * 8)()
    rc = lib.puzzle_unpack(ctypes.cast(buf, ctypes.c_void_p), 0, 8, ctypes.cast(out, ctypes.c_void_p), None)
    assert rc == 5 and b"no CUDA device" in lib.puzzle_last_error()


def test_binding_rejects_cpu_tensors(lib):
    import paper_2511_04805_b200 as pz
    with pytest.raises(ValueError):
        pz.unpack(torch.zeros(8, dtype=torch.int16), 0)


def test_next_row_argument_errors_are_synchronous(lib):
    """NEXT-3 / NEXT-4 entry points reject bad arguments before touching a device."""
    assert lib.puzzle_quant_pack(None, None, None, None, None, 2, 100, None, None, None) == 3   # cols % 128
    assert lib.puzzle_quant_pack(None, None, None, None, None, 2, 128, None, None, None) == 1   # NULL
    assert lib.puzzle_quant_pack(None, None, None, None, None, 0, 128, None, None, None) == 0   # empty: no-op
    assert lib.puzzle_quant_unpack(None, None, 2, 1, 128, None, None) == 1                     # pos
    assert lib.puzzle_quant_unpack(None, None, 0, -1, 128, None, None) == 1                    # negative
    assert lib.puzzle_quant_gemv(None, None, 4, 100, None, 1, None, 0, None, None, None) == 3   # cols % 128
    assert lib.puzzle_quant_gemv(None, None, 4, 128, None, -1, None, 0, None, None, None) == 1  # negative
    assert lib.puzzle_quant_gemv(None, None, 4, 128, None, 1, None, 0, None, None, None) == 1   # NULL
    assert lib.puzzle_quant_gemv(None, None, 4, 128, None, 0, None, 0, None, None, None) == 0   # no tokens: no-op
    assert lib.puzzle_group_colsumsq(None, None, 2, 12, None, None, 0, None) == 1              # NULL
    assert lib.puzzle_group_colsumsq(None, None, 0, 16, None, None, 0, None) == 0              # no groups
    assert lib.puzzle_group_colsumsq_workspace_size(-1, 8) == 0
    import paper_2511_04805_b200 as pz
    desc = pz.MoELayerDesc(8, 4, 4096, 14336, 4096, 4096, 4096)
    assert lib.puzzle_moe_calib_workspace_size(ctypes.byref(desc), 64, 2) > lib.puzzle_moe_workspace_size(
        ctypes.byref(desc), 64, 2)
    # both statistics outputs NULL
    assert lib.puzzle_moe_forward_calib(ctypes.byref(desc), None, None, 1, 2, 1, None, None, None, None, None, 0, 0,
                                        None) == 1


def test_ep_capi_host_side(lib):
    """Expert parallelism behind the C ABI: the placement (puzzle_ep_partition) equals the
    Python partition the gloo tests exercise; the NCCL bootstrap id is 128 bytes; argument
    errors are synchronous; without a device the communicator is refused loudly."""
    import paper_2511_04805_b200 as pz
    from paper_2511_04805_b200.ep import Partition
    for P, G in [(4, 1), (4, 2), (4, 3), (4, 8), (30, 8), (32, 4), (2, 4), (1, 2), (60, 7)]:
        dest, S = pz.ep_partition(G, P)
        part = Partition(P, G)
        assert S == part.slices
        assert dest.tolist() == [list(part.pairs_of(q)) for q in range(G)]
    assert lib.puzzle_ep_partition(8, 3, None, None) == 3            # world > P, world % P != 0
    assert lib.puzzle_ep_partition(0, 4, None, None) == 1
    assert len(pz.ep_unique_id()) == pz.EP_UNIQUE_ID_BYTES
    assert lib.puzzle_moe_forward_ep(None, None, None, None, None, 1, 1, 1, 1, None, None, None, 0, 0, None) == 1
    assert b"handle" in lib.puzzle_last_error()
    assert lib.puzzle_ep_destroy(None) == 0
    assert lib.puzzle_status_string(6) == b"PUZZLE_ERR_NCCL"
    if not torch.cuda.is_available():
        h = ctypes.c_void_p(None)
        assert lib.puzzle_ep_create(ctypes.byref(h), 2, 0, b"\0" * 128, 0) == 5
        assert not h.value

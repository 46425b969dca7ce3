"""The C-ABI library loads and exports every symbol include/msn_pkm.h declares;
host-side validation (no GPU needed: validation runs before any launch)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msn_pkm.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2602_07526_b200 import _build, _lib
    _build.build()
    return _lib.load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msn_pkm_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("msn_pkm_create", "msn_pkm_forward", "msn_pkm_backward", "msn_pkm_destroy"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    from paper_2602_07526_b200 import _lib
    names = declared_functions()
    for n in names:
        assert hasattr(lib, n), f"{n} declared in msn_pkm.h but not exported"
        assert n in _lib.SIGNATURES, f"{n} has no ctypes signature in the binding"


def test_library_has_no_host_fallback_symbols(lib):
    # the product library is CUDA only: it must contain sm_100a device code
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {os.path.join(ROOT, 'paper_2602_07526_b200', 'libmsn_pkm.so')}").read()
    assert "sm_100a" in out


def _cfg(**kw):
    from paper_2602_07526_b200 import _lib
    base = dict(abi_version=2, heads=2, n_sub=64, d_half=32, d_value=64, k=8, max_batch=16,
                qk_dtype=0, value_dtype=0, flags=0, reserved=0, row_begin=0, row_end=64 * 64)
    base.update(kw)
    return _lib.Config(**base)


@pytest.mark.parametrize("bad,status", [
    (dict(abi_version=1), 1), (dict(world_size=9), 1), (dict(world_size=2, rank=2), 1),
    (dict(world_size=3), 1), (dict(world_size=2, row_begin=0, row_end=100), 1), (dict(heads=0), 1), (dict(k=0), 1), (dict(k=65, n_sub=128, row_end=128 * 128), 2),
    (dict(k=70), 1), (dict(d_half=24), 1), (dict(d_value=2, value_dtype=0), 1),
    (dict(row_begin=10, row_end=5), 1), (dict(flags=0x80), 1), (dict(qk_dtype=7), 1),
    (dict(n_sub=4096, row_end=4096 * 4096), 2),
])
def test_create_validates(lib, bad, status):
    h = ctypes.c_void_p()
    s = lib.msn_pkm_create(ctypes.byref(_cfg(**bad)), ctypes.byref(h))
    assert s == status, lib.msn_pkm_last_error()
    assert lib.msn_pkm_last_error()


def test_create_destroy_and_argument_checks(lib):
    h = ctypes.c_void_p()
    assert lib.msn_pkm_create(ctypes.byref(_cfg()), ctypes.byref(h)) == 0
    f, b = ctypes.c_size_t(), ctypes.c_size_t()
    assert lib.msn_pkm_workspace_size(h, 16, 16, ctypes.byref(f), ctypes.byref(b)) == 0
    assert f.value > 0 and b.value > 0
    assert lib.msn_pkm_workspace_size(h, 17, 17, ctypes.byref(f), ctypes.byref(b)) == 1
    # B = 0 is a no-op
    assert lib.msn_pkm_forward(h, None, 0, None, None, None, None, None, None, None, 0) == 0
    # null / misaligned pointers are rejected before any launch
    assert lib.msn_pkm_forward(h, None, 4, None, None, None, None, None, None, None, 0) == 1
    p = ctypes.c_void_p(0x1000)
    mis = ctypes.c_void_p(0x1004)
    assert lib.msn_pkm_forward(h, None, 4, mis, p, p, p, p, p, p, 1 << 30) == 1
    assert b"aligned" in lib.msn_pkm_last_error()
    assert lib.msn_pkm_forward(h, None, 4, p, p, p, p, p, p, p, 16) == 5  # workspace too small
    assert lib.msn_pkm_destroy(h) == 0
    assert lib.msn_pkm_status_string(2) == b"unsupported"


def test_sharded_handle_rejects_full_forward(lib):
    h = ctypes.c_void_p()
    assert lib.msn_pkm_create(ctypes.byref(_cfg(row_begin=0, row_end=2048)), ctypes.byref(h)) == 0
    p = ctypes.c_void_p(0x1000)
    assert lib.msn_pkm_forward(h, None, 4, p, p, p, p, p, p, p, 1 << 30) == 1
    lib.msn_pkm_destroy(h)


def _x(lib_mod, world, rank, lb, transport=0, bases=None):
    x = lib_mod.Exchange()
    x.transport, x.world, x.rank, x.local_batch = transport, world, rank, lb
    for i, b in enumerate(bases or []):
        x.base[i] = b
    return x


def test_sharded_config_and_exchange_checks(lib):
    """world_size > 1 derives the rank's rows [r n/P, (r+1) n/P); the exchange
    calls validate world/rank/transport/bases on the host before any launch."""
    from paper_2602_07526_b200 import _lib
    h = ctypes.c_void_p()
    assert lib.msn_pkm_create(ctypes.byref(_cfg(world_size=4, rank=1, row_begin=0, row_end=0)), ctypes.byref(h)) == 0
    offs = (ctypes.c_int64 * len(_lib.XREG))()
    nb = ctypes.c_size_t()
    assert lib.msn_pkm_exchange_layout(h, 16, 1, offs, ctypes.byref(nb)) == 0
    assert list(offs) == sorted(offs) and all(o % 256 == 0 for o in offs) and nb.value >= offs[-1]
    peer = ctypes.c_size_t()
    assert lib.msn_pkm_exchange_layout(h, 16, 0, None, ctypes.byref(peer)) == 0 and peer.value < nb.value
    # IN_ROW holds P * cap int32 records, cap = B_l * H * k (one window of H * k per query)
    assert offs[1] - offs[0] >= 4 * 4 * 16 * 2 * 8
    p = ctypes.c_void_p(0x100000)
    good = _x(_lib, 4, 1, 16, 0, [0x100000, 0x200000, 0x300000, 0x400000])
    assert lib.msn_pkm_exchange_select(h, None, None, None, None, ctypes.byref(good), None, None, None,
                                       None, 0) == 1     # null query
    for bad in (_x(_lib, 2, 1, 16, 0, [0x100000] * 2), _x(_lib, 4, 0, 16, 0, [0x100000] * 4),
                _x(_lib, 4, 1, 17, 0, [0x100000] * 4), _x(_lib, 4, 1, 16, 5, [0x100000] * 4),
                _x(_lib, 4, 1, 16, 0, [0x100000, 0x100010, 0x100000, 0x100000]),
                _x(_lib, 4, 1, 16, 0, [0x100000, 0, 0x100000, 0x100000])):
        assert lib.msn_pkm_exchange_select(h, None, p, p, p, ctypes.byref(bad), p, p, p, p,
                                           1 << 30) == 1, lib.msn_pkm_last_error()
    # staged: only base[rank] is needed; forward_sharded needs the peer transport
    st = _x(_lib, 4, 1, 16, 1, [0, 0x100000, 0, 0])
    assert lib.msn_pkm_forward_sharded(h, None, 16, p, p, p, ctypes.byref(st), p, p, p, p, 1 << 30) == 1
    assert b"PEER" in lib.msn_pkm_last_error()
    # the whole-table forward is refused on a shard
    assert lib.msn_pkm_forward(h, None, 4, p, p, p, p, p, p, p, 1 << 30) == 1
    lib.msn_pkm_destroy(h)

"""The drop-in boundary: libprescope_b200.so loads and exports every symbol
include/ps_api.h declares (no compute calls — CPU safe)."""
import ctypes as C
import subprocess

import numpy as np

import paper_2509_23638_b200 as ps
from conftest import ROOT


def test_library_exports_every_declared_symbol():
    declared = ps.capi.declared_symbols()
    assert len(declared) >= 40
    lib = ps.load()
    missing = [s for s in declared if not hasattr(lib, s)]
    assert missing == [], missing
    out = subprocess.run(["nm", "-D", "--defined-only", str(ps.capi.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_every_declared_symbol_has_a_ctypes_signature():
    assert set(ps.capi.declared_symbols()) <= set(ps.capi._SIGS)


def test_version_and_error_channel():
    lib = ps.load()
    assert b"sm_100a" in lib.ps_version()
    spec = ps.capi.ModelSpec()
    assert lib.ps_spec_preset(b"nope", C.byref(spec)) == ps.capi.PS_EINVAL
    assert b"unknown model preset" in lib.ps_last_error()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(ps.capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_product_does_not_import_oracle():
    for p in (ROOT / "paper_2509_23638_b200").rglob("*.py"):
        text = p.read_text()
        assert "import oracle" not in text and "from oracle" not in text, p


def test_argument_validation_before_any_launch():
    """Entry points reject bad shapes with PS_EINVAL before touching the GPU (CPU safe)."""
    lib = ps.load()
    assert lib.ps_set_prefill_kernel(4) == ps.capi.PS_EINVAL
    assert lib.ps_set_prefill_kernel(2) == ps.capi.PS_OK
    # fused route+permute is a decode-only launch: B <= 64
    p = C.c_void_p(16)
    assert lib.ps_route_permute(p, p, None, None, None, 2, 65, 64, 8, 2, p, p, p, p, p, p, p, None) == ps.capi.PS_EINVAL
    assert b"decode shapes only" in lib.ps_last_error()
    # z-slab codec: null / empty arguments
    nb = C.c_uint64()
    assert lib.ps_zslab_encode(None, 0, None, 0, C.byref(nb), 1) == ps.capi.PS_EINVAL
    assert lib.ps_zslab_bound(1024) > 1024
    # shared-expert append: S out of range
    assert lib.ps_append_shared(p, p, 4, 2, 8, 0, p, p, None, None) == ps.capi.PS_EINVAL
    # K3 on z-slabs: shape / token-count checks, and an all-idle group is a no-op (no launch)
    grp = ps.capi.ExpertGroup()
    grp.n = 2
    grp.experts[0], grp.experts[1] = 0, 1
    zp = (C.c_void_p * 2)(16, 32)
    idle = np.zeros(2, np.int32)
    assert lib.ps_expert_ffn_zslab(C.byref(grp), zp, idle.ctypes.data, p, p, 1, p, 256, 512, p, p, 1, 8,
                                   None) == ps.capi.PS_OK
    busy = np.array([9, 0], np.int32)
    assert lib.ps_expert_ffn_zslab(C.byref(grp), zp, busy.ctypes.data, p, p, 1, p, 256, 512, p, p, 1, 9,
                                   None) == ps.capi.PS_EINVAL
    assert b"8 tokens" in lib.ps_last_error()
    assert lib.ps_expert_ffn_zslab(C.byref(grp), zp, idle.ctypes.data, p, p, 1, p, 96, 512, p, p, 1, 8,
                                   None) == ps.capi.PS_EINVAL
    assert lib.ps_expert_ffn_zslab(C.byref(grp), None, idle.ctypes.data, p, p, 1, p, 256, 512, p, p, 1, 8,
                                   None) == ps.capi.PS_EINVAL

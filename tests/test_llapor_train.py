"""Online LLaPor fine_tune (predictor.cpp:654-663) and LLPC save (predictor.cpp:833-875)
of the product (ps_llapor_fine_tune / ps_llapor_save, host f64) vs the UNMODIFIED
reference (oracle/_ref): the fine-tuned model saved by both must be byte-identical —
every weight, bias, gate and AdamW-updated parameter bit for bit. CPU only (the GPU copy
of a net is refreshed lazily before its next forward)."""
import ctypes as C

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps
from conftest import GOLDEN
from oracle.llpc import random_nets, write_llpc

pytestmark = pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")


def _load(path):
    m = C.c_void_p()
    spec = ps.capi.ModelSpec()
    ps.check(ps.load().ps_llapor_load(str(path).encode(), C.byref(m), C.byref(spec)))
    return m, spec


def test_save_round_trips_reference_checkpoint_bytes(tmp_path):
    """A reference-trained checkpoint (tests/golden/llapor_desk.llpc) re-saved by the
    product is byte-identical: every field of save_checkpoint is kept."""
    m, _ = _load(GOLDEN / "llapor_desk.llpc")
    try:
        out = tmp_path / "resaved.llpc"
        ps.check(ps.load().ps_llapor_save(m, str(out).encode()))
        assert out.read_bytes() == (GOLDEN / "llapor_desk.llpc").read_bytes()
    finally:
        ps.load().ps_llapor_free(m)


def _samples(spec, B, seed, layer):
    """build_samples pairs from a reference trace: features of layer-1, labels of layer."""
    rg = orc.ref_gen(*[ps.GROUP_DEFAULT_GEN[g] for g in ("input", "middle", "output")])
    hidden, gw, act = orc.ref_trace(rg, orc.ref_spec_from(spec), B, seed)
    return (np.ascontiguousarray(hidden[:, layer - 1]), np.ascontiguousarray(act[:, layer - 1]),
            np.ascontiguousarray(gw[:, layer - 1]), np.ascontiguousarray(act[:, layer]))


def _fine_tune_both(path, spec, layers, B, steps, lr, tmp_path):
    lib, ref = ps.load(), orc.ref_lib()
    m, _ = _load(path)
    h = ref.ref_llapor_load(str(path).encode())
    assert h
    try:
        for layer in layers:
            hid, ap, gp, a = _samples(spec, B, 100 + layer, layer)
            k = a.shape[1]
            args = (layer, B, hid.ctypes.data, ap.ctypes.data, ap.shape[1], gp.ctypes.data, a.ctypes.data, k, steps, lr)
            ps.check(lib.ps_llapor_fine_tune(m, *args))
            orc.ref_check(ref.ref_llapor_fine_tune(h, *args))
        mine, theirs = tmp_path / "mine.llpc", tmp_path / "theirs.llpc"
        ps.check(lib.ps_llapor_save(m, str(mine).encode()))
        orc.ref_check(ref.ref_llapor_save(h, str(theirs).encode()))
        before = pathlib_bytes(path)
        assert mine.read_bytes() != before, "fine_tune changed nothing"
        assert mine.read_bytes() == theirs.read_bytes()
    finally:
        lib.ps_llapor_free(m)
        ref.ref_llapor_free(h)


def pathlib_bytes(p):
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.parametrize("steps,lr", [(1, 1e-3), (4, 3e-3)])
def test_fine_tune_reference_trained_desk_model_bit_exact(tmp_path, steps, lr):
    """Desk config (BASELINE config[0]): the reference-trained model fine-tuned on fresh
    reference-trace samples for every net (input, middle with gated residual, output)."""
    spec = ps.desk_scale("mixtral", 4, 8, 16)
    _fine_tune_both(GOLDEN / "llapor_desk.llpc", spec, [1, 2, 3], 48, steps, lr, tmp_path)


def test_fine_tune_full_shape_bit_exact(tmp_path):
    """Paper dims: P=512 over H=4096 (middle net), P=256 (output net), E=8, 40 samples
    (two minibatches of 32: the second is ragged)."""
    spec = ps.desk_scale("mixtral", 3, 8, 4096)
    path = tmp_path / "full.llpc"
    write_llpc(path, spec, random_nets(spec, 256, 512, 32, 48, seed=3))
    _fine_tune_both(path, spec, [1, 2], 40, 2, 1e-3, tmp_path)


def test_random_model_saves_what_the_reference_reads(tmp_path):
    """ps_llapor_random -> ps_llapor_save -> the reference's load_checkpoint +
    save_checkpoint reproduces the file (the writer follows save_checkpoint's layout)."""
    lib = ps.load()
    spec = ps.desk_scale("qwen3", 4, 128, 256)
    m = C.c_void_p()
    ps.check(lib.ps_llapor_random(C.byref(spec), 32, 64, 32, 48, 5, C.byref(m)))
    try:
        a = tmp_path / "a.llpc"
        ps.check(lib.ps_llapor_save(m, str(a).encode()))
    finally:
        lib.ps_llapor_free(m)
    h = orc.ref_lib().ref_llapor_load(str(a).encode())
    assert h
    b = tmp_path / "b.llpc"
    orc.ref_check(orc.ref_lib().ref_llapor_save(h, str(b).encode()))
    orc.ref_lib().ref_llapor_free(h)
    assert a.read_bytes() == b.read_bytes()


def test_fine_tune_argument_errors():
    lib = ps.load()
    m, _ = _load(GOLDEN / "llapor_desk.llpc")
    try:
        x = np.zeros((2, 16))
        ids = np.zeros((2, 2), np.int32)
        gw = np.full((2, 8), 0.125)
        assert lib.ps_llapor_fine_tune(m, 0, 2, x.ctypes.data, ids.ctypes.data, 2, gw.ctypes.data, ids.ctypes.data,
                                       2, 1, 1e-3) == ps.capi.PS_ERANGE  # nets[0] is untrained
        bad = np.full((2, 2), 9, np.int32)
        assert lib.ps_llapor_fine_tune(m, 1, 2, x.ctypes.data, bad.ctypes.data, 2, gw.ctypes.data, ids.ctypes.data,
                                       2, 1, 1e-3) == ps.capi.PS_ERANGE
    finally:
        lib.ps_llapor_free(m)

"""Trace file format v1 (write_trace / read_trace, workload.cpp:290-436) — SURVEY.md
§8f row 1: the product reads traces the reference wrote and writes byte-identical ones.

Pinned by tests/golden/ref_trace_desk.tsv (written by the unmodified reference, see
make_golden.py) and, when oracle/_ref is built, by fresh reference traces of the three
SURVEY §8c fingerprint configs (their FNV-1a checksums are in trace_fingerprints.json)."""
import ctypes as C
import json
import pathlib

import numpy as np
import pytest

import oracle as orc
import paper_2509_23638_b200 as ps

GOLD = pathlib.Path(__file__).parent / "golden"


def test_fnv1a64_constants():
    lib = ps.load()
    # test_workload.cpp:238-242: empty string -> offset basis; "a" -> 0xaf63dc4c8601ec8c
    assert lib.ps_fnv1a64(None, 0) == 0xcbf29ce484222325
    assert lib.ps_fnv1a64(b"a", 1) == 0xaf63dc4c8601ec8c


def test_read_reference_trace_and_rewrite_byte_identical(tmp_path):
    t = ps.read_trace(GOLD / "ref_trace_desk.tsv")
    s = t.spec
    assert (s.num_layers, s.experts_per_layer, s.top_k, s.hidden_dim) == (4, 8, 2, 16)
    assert (t.batch_size, t.seed) == (3, 17)
    # trace invariants (test_workload.cpp:92-120)
    np.testing.assert_allclose(t.gate_weights.sum(-1), 1.0, rtol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(t.hidden, axis=-1), 1.0, rtol=1e-12)
    for b in range(3):
        for l in range(4):
            w = t.gate_weights[b, l]
            top = np.zeros(2, np.int32)
            ps.load().ps_topk_indices(w.ctypes.data_as(C.c_void_p), 8, 2, top.ctypes.data_as(C.c_void_p))
            assert top.tolist() == t.active[b, l].tolist()
            assert t.tokens[b, l].sum() == 2 and all(t.tokens[b, l, e] == 1 for e in top)
    out = tmp_path / "re.tsv"
    ps.write_trace(t, out)
    assert out.read_bytes() == (GOLD / "ref_trace_desk.tsv").read_bytes()
    # header checksum = FNV-1a of the body
    body = out.read_bytes().split(b"\n", 1)[1]
    assert ps.load().ps_fnv1a64(body, len(body)) == t.checksum


def _expect_error(path, needle):
    with pytest.raises(ps.capi.PsError) as ei:
        ps.read_trace(path)
    assert needle in str(ei.value)
    return ei.value


def test_checksum_and_format_errors(tmp_path):
    raw = (GOLD / "ref_trace_desk.tsv").read_bytes()
    head, body = raw.split(b"\n", 1)
    # flip one digit in the body -> TraceChecksumError (runtime_error)
    i = body.index(b"0.", 10) + 3
    bad = bytearray(body)
    bad[i] = ord("1") if bad[i] != ord("1") else ord("2")
    p = tmp_path / "cs.tsv"
    p.write_bytes(head + b"\n" + bytes(bad))
    assert _expect_error(p, "TraceChecksumError").status == ps.capi.PS_ERUNTIME
    # unsupported version / bad header / wrong field count -> TraceFormatError
    p.write_bytes(head.replace(b'"format_version":1', b'"format_version":2') + b"\n" + body)
    _expect_error(p, "unsupported format version")
    p.write_bytes(b"{not json\n" + body)
    _expect_error(p, "TraceFormatError")
    p.write_bytes(b"")
    _expect_error(p, "missing header")
    lines = body.split(b"\n")
    lines[0] = lines[0].rsplit(b"\t", 1)[0]
    p.write_bytes(head + b"\n" + b"\n".join(lines))
    _expect_error(p, "expected 5 fields")
    _expect_error(tmp_path / "absent.tsv", "cannot open")


def test_invalid_spec_in_header_is_invalid_argument(tmp_path):
    raw = (GOLD / "ref_trace_desk.tsv").read_bytes()
    p = tmp_path / "spec.tsv"
    p.write_bytes(raw.replace(b'"top_k":2', b'"top_k":9', 1))
    with pytest.raises(ps.capi.PsError) as ei:
        ps.read_trace(p)
    assert ei.value.status == ps.capi.PS_EINVAL


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_reference_traces_roundtrip_and_fingerprints(tmp_path):
    """Fresh reference traces of the SURVEY §8c configs: our reader recovers the
    reference's arrays, our writer reproduces its bytes, checksums match the pinned
    fingerprints."""
    fps = json.loads((GOLD / "trace_fingerprints.json").read_text())
    for fp in fps:
        name, L, E, H = fp["spec"]
        spec = ps.desk_scale(name, L, E, H)
        gen = orc.ref_gen(*([tuple(fp["knobs"])] * 3))
        p = tmp_path / "ref.tsv"
        orc.ref_check(orc.ref_lib().ref_write_trace(C.byref(gen), C.byref(orc.ref_spec_from(spec)), fp["batch"],
                                                    fp["seed"], str(p).encode()))
        t = ps.read_trace(p)
        assert t.checksum == int(fp["fnv1a"])
        hid, gw, act = orc.ref_trace(gen, orc.ref_spec_from(spec), fp["batch"], fp["seed"])
        np.testing.assert_array_equal(t.hidden.reshape(hid.shape), hid)
        np.testing.assert_array_equal(t.gate_weights.reshape(gw.shape), gw)
        np.testing.assert_array_equal(t.active.reshape(act.shape), act)
        q = tmp_path / "ours.tsv"
        ps.write_trace(t, q)
        assert q.read_bytes() == p.read_bytes()


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_reference_reads_our_trace(tmp_path):
    """The other direction: a file written by ps_trace_write (here from modified arrays,
    so it is not a byte copy of a reference file) is accepted by the reference's
    read_trace (checksum, header) and parses to the same routing."""
    t = ps.read_trace(GOLD / "ref_trace_desk.tsv")
    t.seed = 99
    t.active = t.active[:, :, ::-1].copy()  # any routing: the reader does not re-derive it
    p = tmp_path / "ours.tsv"
    ps.write_trace(t, p)
    b, seed = C.c_int(), C.c_uint64()
    act = np.zeros(t.active.size, np.int32)
    orc.ref_check(orc.ref_lib().ref_read_trace(str(p).encode(), C.byref(b), C.byref(seed), act.ctypes.data, act.size))
    assert (b.value, seed.value) == (t.batch_size, 99)
    np.testing.assert_array_equal(act, t.active.ravel())


def test_semantic_errors_after_checksum(tmp_path):
    """Files the reference would parse but a dense trace cannot hold (extra hidden value,
    expert id >= E) raise TraceFormatError when their checksum is valid, and
    TraceChecksumError when it is not (the reference checks the checksum after parsing)."""
    lib = ps.load()
    raw = (GOLD / "ref_trace_desk.tsv").read_bytes()
    head, body = raw.split(b"\n", 1)
    lines = body.split(b"\n")
    f = lines[0].split(b"\t")
    f[1] = f[1] + b" 0.5"
    lines[0] = b"\t".join(f)
    nb = b"\n".join(lines)
    hdr = json.loads(head)
    hdr["checksum"] = lib.ps_fnv1a64(nb, len(nb))
    good_head = json.dumps(hdr, separators=(",", ":"), sort_keys=True).encode()
    p = tmp_path / "sem.tsv"
    p.write_bytes(good_head + b"\n" + nb)
    _expect_error(p, "too many hidden")
    p.write_bytes(head + b"\n" + nb)  # stale checksum
    _expect_error(p, "TraceChecksumError")

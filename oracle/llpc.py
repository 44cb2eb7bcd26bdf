"""TEST / BASELINE INFRASTRUCTURE (tests and bench.py's CPU-baseline arm only): random LLaPor nets at full paper shapes written as LLPC v1 checkpoints
(the layout of save_checkpoint, predictor.cpp:833-875), so the GPU loader/kernel
(ps_llapor_load + ps_llapor_forward) and the reference's own load_checkpoint + forward
(oracle/_ref) read the SAME weights. Net structure follows make_llapor / TrainConfig
defaults (predictor.cpp:473-520, predictor.hpp:97-100): input/output groups 2 GELU
blocks of width w_in, the middle group 3 blocks of width w_mid + 2 residual blocks and
a PCA-space gate; nets[0] is untrained (no blocks)."""
from __future__ import annotations

import struct

import numpy as np


def _dims(spec):
    """(L, E, k, H, expert_bytes, group_begin_middle, group_begin_output) of a product
    ModelSpec or an oracle RefSpec."""
    E = getattr(spec, "experts_per_layer", None) or spec.experts
    H = getattr(spec, "hidden_dim", None) or spec.hidden
    return (spec.num_layers, E, spec.top_k, H, spec.expert_bytes, spec.group_begin_middle, spec.group_begin_output)


def group_of(spec, layer):
    return 0 if layer < spec.group_begin_middle else (1 if layer < spec.group_begin_output else 2)


def random_nets(spec, p_in, p_mid, w_in, w_mid, seed):
    """-> list of nets (index = target layer; nets[0] = None)."""
    rng = np.random.default_rng(seed)
    L, E, _, H = _dims(spec)[:4]
    nets = [None]
    for l in range(1, L):
        g = group_of(spec, l)
        P, width, nb = (p_mid, w_mid, 3) if g == 1 else (p_in, w_in, 2)
        P = min(P, H)

        def xavier(o, i):
            a = np.sqrt(6.0 / (i + o))
            return rng.uniform(-a, a, (o, i)), rng.uniform(-0.05, 0.05, o)

        comp = rng.standard_normal((P, H)) / np.sqrt(H)
        blocks, d = [], P + 2 * E
        for _ in range(nb):
            blocks.append(xavier(width, d))
            d = width
        res = [xavier(width, width) for _ in range(2)] if g == 1 else []
        gate_w = rng.uniform(-0.1, 0.1, P) if g == 1 else np.zeros(0)
        nets.append({"target": l, "group": g, "E": E, "mean": rng.standard_normal(H) * 0.01, "comp": comp,
                     "blocks": blocks, "res": res, "gate_w": gate_w, "gate_b": 0.05, "out": xavier(E, width)})
    return nets


def write_llpc(path, spec, nets, trace_checksum=0):
    out = bytearray(b"LLPC")

    def w(fmt, *v):
        out.extend(struct.pack("<" + fmt, *v))

    def vec(a):
        a = np.ascontiguousarray(a, np.float64).ravel()
        w("Q", a.size)
        out.extend(a.tobytes())

    def mat(a):
        a = np.atleast_2d(np.asarray(a, np.float64))
        w("ii", a.shape[0], a.shape[1])
        vec(a)

    def block(b):
        mat(b[0])
        vec(b[1])

    L, E, k, H, eb, gbm, gbo = _dims(spec)
    w("I", 1)
    w("Q", trace_checksum)
    w("iii", L, E, k)
    w("Q", eb)
    w("iii", H, gbm, gbo)
    w("dd", 0.0, 0.0)       # lambda, gamma
    w("ii", 0, 0)           # epochs, warmup
    for _ in range(3):
        w("ddiii", 1e-3, 0.0, 0, 0, 0)
    w("ddd", 0.0, 0.0, 0.0)  # dropout, noise, mask
    w("i", 1)
    w("Q", 0)
    w("I", len(nets))
    for l, n in enumerate(nets):
        if n is None:  # untrained nets[0]
            w("iBid", 0, 0, E, 0.0)
            vec([])
            w("ii", 0, 0)
            vec([])
            vec([])
            w("ii", 0, 0)
            w("I", 0)
            w("I", 0)
            vec([])
            w("d", 0.0)
            w("ii", 0, 0)
            vec([])
            vec([])
            continue
        w("iBid", n["target"], n["group"], n["E"], 0.0)
        vec(n["mean"])
        mat(n["comp"])
        vec(np.ones(n["comp"].shape[0]))  # eigenvalues (unused by inference)
        w("ii", n["comp"].shape[0], n["comp"].shape[0])
        w("I", len(n["blocks"]))
        for b in n["blocks"]:
            block(b)
        w("I", len(n["res"]))
        for b in n["res"]:
            block(b)
        vec(n["gate_w"])
        w("d", n["gate_b"])
        block(n["out"])
    with open(path, "wb") as f:
        f.write(bytes(out))

"""Run-to-run determinism stress of K3 decode (ps_expert_ffn): the kernel is
deterministic by construction, so any bitwise difference between repeats exposes a race.
Reports which permuted rows / experts / outputs (h or y_part) differ.

  python scripts/ffn_stress.py --H 2048 --F 768 --E 128 --k 8 --B 32 --reps 50
"""
import argparse
import ctypes as C
import pathlib
import sys

import numpy as np
import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2509_23638_b200 as ps  # noqa: E402


SYNC_AFTER_INIT = False
TOUCH = False


def _p(t):
    return C.c_void_p(t.data_ptr())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=2048)
    ap.add_argument("--F", type=int, default=768)
    ap.add_argument("--E", type=int, default=128)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--B", type=int, default=32)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--sync-after-init", action="store_true")
    ap.add_argument("--touch", action="store_true")
    a = ap.parse_args()
    global SYNC_AFTER_INIT, TOUCH
    SYNC_AFTER_INIT = a.sync_after_init
    TOUCH = a.touch
    lib = ps.load()
    H, F, E, k, B = a.H, a.F, a.E, a.k, a.B
    rng = np.random.default_rng(a.seed)
    ids = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
    s = torch.cuda.current_stream()
    sp = C.c_void_p(s.cuda_stream)
    slabs = [torch.empty(3 * H * F, dtype=torch.int16, device="cuda") for _ in range(E)]
    for e in range(E):
        ps.check(lib.ps_init_expert_slab(_p(slabs[e]), H, F, 1, 0, e, sp))
    if SYNC_AFTER_INIT:
        torch.cuda.synchronize()
    if TOUCH:
        tot = sum(float(sl.float().sum()) for sl in slabs)  # warm TLB / page tables
        print("touched", tot != 0)
    di = torch.as_tensor(ids, device="cuda")
    off = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    src = torch.empty(B * k, dtype=torch.int32, device="cuda")
    inv = torch.empty(B * k, dtype=torch.int32, device="cuda")
    ps.check(lib.ps_permute(_p(di), B, k, E, _p(off), _p(src), _p(inv), None, H, None, sp))
    n_split = lib.ps_ffn_down_splits(H, F)
    x = (torch.randn(B, H, device="cuda") / H ** 0.5).to(torch.bfloat16).view(torch.int16)
    counts = np.bincount(ids.ravel(), minlength=E).astype(np.int32)
    grp = ps.capi.ExpertGroup()
    grp.n = E
    for e in range(E):
        grp.experts[e] = e
        grp.slabs[e] = slabs[e].data_ptr()
    offs = off.cpu().numpy()
    ref_h = ref_y = None
    bad = 0
    for r in range(a.reps):
        h = torch.full((B * k, F), -1, dtype=torch.int16, device="cuda")
        yp = torch.full((n_split, B * k, H), float("nan"), dtype=torch.float32, device="cuda")
        ps.check(lib.ps_expert_ffn(C.byref(grp), counts.ctypes.data, _p(off), _p(src), k, _p(x), H, F, _p(h), _p(yp),
                                   n_split, B * k, sp))
        torch.cuda.synchronize()
        hh, yy = h.cpu().numpy(), yp.cpu().numpy()
        # down-phase check from the kernel's own h: y_part[s] = Wd[:, split s] . h[split s]
        kch = ((F + n_split - 1) // n_split + 31) // 32 * 32
        worst = 0.0
        for e in range(E):
            r0, r1 = int(offs[e]), int(offs[e + 1])
            if r1 == r0:
                continue
            wd = slabs[e][2 * F * H:].view(torch.bfloat16).view(H, F).float()
            he = h[r0:r1].view(torch.bfloat16).float()
            for sp_ in range(n_split):
                b, c = min(F, sp_ * kch), min(F, sp_ * kch + kch)
                ref = he[:, b:c] @ wd[:, b:c].T
                d = (yp[sp_, r0:r1] - ref).abs()
                err = d.max().item() / max(ref.abs().max().item(), 1e-30)
                worst = max(worst, err)
                if err > 1e-3 and r == 0:
                    bad_d = torch.nonzero(d.max(0).values > 1e-3 * ref.abs().max()).flatten().tolist()
                    print(f"   rep0 expert {e} split {sp_} err {err:.2e} bad d {len(bad_d)}: {bad_d[:6]}..{bad_d[-3:]}")
        print(f"rep {r}: down-phase max rel err vs own h = {worst:.2e}")
        if ref_h is None:
            ref_h, ref_y = hh, yy
            continue
        dh = np.argwhere(hh != ref_h)
        dy = np.argwhere(~((yy == ref_y) | (np.isnan(yy) & np.isnan(ref_y))))
        if len(dh) or len(dy):
            bad += 1
            rows_h = sorted(set(dh[:, 0].tolist()))
            rows_y = sorted(set(dy[:, 1].tolist()))
            exp_of = lambda row: int(np.searchsorted(offs, row, side="right") - 1)  # noqa: E731
            print(f"rep {r}: h diffs {len(dh)} rows {rows_h[:8]} experts {[exp_of(x) for x in rows_h[:8]]}; "
                  f"y diffs {len(dy)} rows {rows_y[:8]} experts {[exp_of(x) for x in rows_y[:8]]} "
                  f"cols {sorted(set(dy[:, 2].tolist()))[:8]}")
            if len(dy):
                sp_, r1, c1 = dy[0]
                print(f"   y[{sp_},{r1},{c1}] ref {ref_y[sp_, r1, c1]} now {yy[sp_, r1, c1]}; splits {sorted(set(dy[:, 0].tolist()))}")
            if len(dh):
                r0, c0 = dh[0]
                print(f"   h[{r0},{c0}] ref {ref_h[r0, c0]} now {hh[r0, c0]}; h diff cols {sorted(set(dh[:, 1].tolist()))[:16]}")
    print(f"{bad} of {a.reps - 1} repeats differ")


if __name__ == "__main__":
    main()

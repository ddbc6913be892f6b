#!/usr/bin/env python
"""Debug: per-warp globaltimer spans of one GEMV launch (FLEXQ_GEMV_TIMELINE=1).

    python tools/gemv_timeline.py N K M [repeats]

Prints the phase summary of the last launch, the per-CTA loop times, and -- over
``repeats`` launches -- the streaming rate of every SM (units per microsecond of its
warps' loops), its run-to-run stability and how it clusters by SM id, to tell a
per-SM bandwidth difference from scheduling noise.
"""
import ctypes
import os
import sys

os.environ["FLEXQ_GEMV_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def grab(lay, m, out):
    import numpy as np
    import torch

    from paper_2508_04405_b200 import _lib

    lay.gemm_only(m, out)
    torch.cuda.synchronize()
    nall = 148 * 16 * 8
    buf = (ctypes.c_longlong * nall)()
    fn = _lib.lib().flexq_debug_gemv_timeline
    fn.restype = ctypes.c_int
    fn(buf, nall)
    a = np.frombuffer(buf, dtype=np.int64).reshape(-1, 8).copy()
    return a[a[:, 0] > 0]


def per_sm(a, units_per_warp):
    """{smid: units per us of loop time, summed over the SM's warps}."""
    import numpy as np
    out = {}
    for sm in np.unique(a[:, 6]):
        rows = a[a[:, 6] == sm]
        dur = (rows[:, 5] - rows[:, 4]) / 1e3
        out[int(sm)] = float(np.sum(units_per_warp / np.maximum(dur, 1e-3)))
    return out


def main():
    import numpy as np
    import torch

    from paper_2508_04405_b200 import FlexQLinear

    args = [int(v) for v in sys.argv[1:]]
    n, k, m = args[:3] if len(args) >= 3 else (4096, 4096, 1)
    reps = args[3] if len(args) > 3 else 4
    lay = FlexQLinear(torch.randn((n, k), device="cuda", dtype=torch.float16), 6, 6, 128)
    x = torch.randn((m, k), device="cuda", dtype=torch.float16)
    out = torch.empty((m, n), device="cuda", dtype=torch.float16)
    for _ in range(3):
        lay.forward(x, out=out)
    torch.cuda.synchronize()
    runs = [grab(lay, m, out) for _ in range(reps)]
    a = runs[-1]
    t0 = a[:, 0].min()
    d = (a[:, [0, 1, 2, 3, 4, 5, 7]] - t0) / 1e3
    print(f"{n}x{k} m={m}: warps {len(a)}, SMs {len(np.unique(a[:, 6]))}")
    for i, name in enumerate(["start", "init_done", "prologue", "pdl_done", "first_data",
                              "loop_done", "end"]):
        print(f"  {name:10s} min {d[:, i].min():7.2f}  median {np.median(d[:, i]):7.2f}  "
              f"max {d[:, i].max():7.2f} us")
    per_cta(a)
    units = (n // 64) * (k // 128) / len(a)
    rates = [per_sm(r, units) for r in runs]
    sms = sorted(rates[0])
    mat = np.array([[r.get(s, np.nan) for s in sms] for r in rates])
    mean = np.nanmean(mat, 0)
    print(f"  per-SM rate (units/us): mean {mean.mean():.2f}, min {mean.min():.2f}, "
          f"max {mean.max():.2f}, cv {mean.std() / mean.mean():.3f}")
    if len(runs) > 1:
        cc = np.corrcoef(mat[0], mat[1])[0, 1]
        print(f"  run-to-run correlation of per-SM rates: {cc:.2f} (1 = fixed per-SM speed)")
    order = np.argsort(mean)
    print("  slowest SMs: " + " ".join(f"{sms[i]}:{mean[i]:.1f}" for i in order[:12]))
    print("  fastest SMs: " + " ".join(f"{sms[i]}:{mean[i]:.1f}" for i in order[-12:]))
    # rate by smid bands of 8 (TPC pairs / GPC neighbourhoods)
    band = {}
    for s, v in zip(sms, mean):
        band.setdefault(s // 16, []).append(v)
    print("  by smid/16: " + " ".join(f"{b}:{np.mean(v):.2f}" for b, v in sorted(band.items())))
    # within each SM: loop end by the CTA's rank among the SM's CTAs (0 = lowest index)
    cta = np.arange(len(a)) // 4
    ranks = {}
    for sm in np.unique(a[:, 6]):
        idx = np.nonzero(a[:, 6] == sm)[0]
        ctas = sorted(set(cta[idx].tolist()))
        for rk, c in enumerate(ctas):
            sel = idx[cta[idx] == c]
            ranks.setdefault(rk, []).append(float(np.mean(a[sel, 5] - t0) / 1e3))
    print("  loop end by CTA rank on its SM: " + " ".join(
        f"r{rk}:{np.mean(v):.2f}(n={len(v)})" for rk, v in sorted(ranks.items())))
    ws = (a[:, 5] - t0) / 1e3
    wr = np.arange(len(a)) % 4
    print("  loop end by warp slot in CTA: " + " ".join(f"w{w}:{ws[wr == w].mean():.2f}" for w in range(4)))
    np.save(os.path.join("gpurun_out", f"gemv_sm_rates_{n}x{k}_m{m}.npy"), np.vstack([sms, mat]))


def per_cta(a, warps_per_cta=4):
    import numpy as np
    dur = (a[:, 5] - a[:, 4]) / 1e3
    n = len(dur) // warps_per_cta * warps_per_cta
    c = dur[:n].reshape(-1, warps_per_cta).mean(1)
    print("  per-CTA loop us: " + " ".join(f"{v:.1f}" for v in c[:48]))
    print(f"  corr(cta index, dur) = {np.corrcoef(np.arange(len(c)), c)[0, 1]:.2f}; "
          f"odd/even CTA mean {c[1::2].mean():.2f}/{c[0::2].mean():.2f}")


if __name__ == "__main__":
    main()

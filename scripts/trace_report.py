"""Summarise an FGA_TRACE timeline (development aid): python scripts/trace_report.py trace.txt"""
import sys

import numpy as np

lines = open(sys.argv[1]).read().split("\n")
t = np.array([[int(x) for x in l.split()] for l in lines[:64]], dtype=np.int64)
tt = np.array([[int(x) for x in l.split()] for l in lines[64:96]], dtype=np.int64)
cta = np.array([[int(x) for x in l.split()] for l in lines[96:96 + 1024] if l.strip()], dtype=np.int64)
wl = [l for l in lines[96 + 1024:96 + 1024 + 64] if l.strip()]
warp_arrive = np.array([[int(x) for x in l.split()] for l in wl], dtype=np.int64) if wl else None
mm = t[:, 8] > 0
j = np.nonzero(mm)[0]
r = j[(j >= 4) & (j < j.max() - 2)]
print("chunks traced", len(j), "MMA period per chunk (S issue)", (np.diff(t[r, 14]) / np.diff(r)).mean())
print(" mma: waitK", (t[r, 9] - t[r, 8]).mean(), "fence", (t[r, 13] - t[r, 9]).mean(), "S issue+commit",
      (t[r, 14] - t[r, 13]).mean())
print(" mma: waitP", (t[r, 11] - t[r, 10]).mean(), "PV(wait V+fence+issue+commit)", (t[r, 12] - t[r, 11]).mean())
if (t[r, 6] > 0).all() and (t[r, 7] > 0).all():
    print("   PV: wait V", (t[r, 6] - t[r, 11]).mean(), "wait PV_{c-1} issued", (t[r, 7] - t[r, 6]).mean(),
          "issue+commit", (t[r, 12] - t[r, 7]).mean(), "| S: wait K", (t[r, 9] - t[r, 8]).mean(),
          "issue+commit", (t[r, 14] - t[r, 9]).mean())
sm = np.nonzero(t[:, 0] > 0)[0]
s = sm[(sm >= 4) & (sm < sm.max() - 2)]
print(" softmax(wg0) chunks", len(sm), "period per chunk", (np.diff(t[s, 5]) / np.diff(s)).mean() if len(s) > 1 else 0)
print(" softmax: waitS", (t[s, 1] - t[s, 0]).mean(), "ld", (t[s, 2] - t[s, 1]).mean(), "max",
      (t[s, 3] - t[s, 2]).mean(), "exp", (t[s, 4] - t[s, 3]).mean(), "st", (t[s, 5] - t[s, 4]).mean())

# tile level (CTA 0): 0 Q issue, 1 MMA got Q, 2 MMA got o_empty (first PV), 3 MMA tile done, 4 epilogue start, 5 epilogue end
v = tt[:, 1] > 0
if v.any():
    k = np.nonzero(v)[0]
    print("tiles (CTA 0)", len(k), "tile period", np.diff(tt[k, 1]).mean() if len(k) > 1 else 0)
    print(" per tile: Qissue->MMA got Q", (tt[k, 1] - tt[k, 0]).mean(), " MMA got Q->o_empty", (tt[k, 2] - tt[k, 1]).mean(),
          " epilogue", (tt[k, 5] - tt[k, 4]).mean(), " lastPV issued->epi start", (tt[k, 4] - tt[k, 3]).mean())
c = cta[cta[:, 0] > 0]
if len(c):
    t0 = c[:, 0].min()
    d = (c[:, 1] - c[:, 0]) / 1e3
    print(f"CTAs {len(c)}: start spread {(c[:, 0].max() - t0) / 1e3:.1f} us, duration min {d.min():.1f} "
          f"median {np.median(d):.1f} max {d.max():.1f} us, end spread {(c[:, 1].max() - c[:, 1].min()) / 1e3:.1f} us")

if warp_arrive is not None and (warp_arrive[:, :8] > 0).all(axis=1).any():
    rows = [r for r in range(4, len(warp_arrive) - 2) if (warp_arrive[r, :8] > 0).all()]
    lag = np.array([warp_arrive[r, :8] - warp_arrive[r, :8].min() for r in rows])
    print(" softmax warp arrive lag behind the first warp (cycles), per warp 0..7:", lag.mean(0).round(0).tolist())

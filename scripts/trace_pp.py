"""Timeline report for the ping-pong kernel's trace build (FGA_ATTN_KERNEL=pp, FGA_TRACE_ON=1)."""
import sys

import numpy as np

rows = [list(map(int, l.split())) for l in open(sys.argv[1]).read().strip().split("\n")]
ch = np.array(rows[:64], dtype=np.int64)
tl = np.array(rows[64:96], dtype=np.int64)
n = int((ch[:, 8] > 0).sum())
t0 = ch[0, 8]
print("chunk: issuer[waitK->gotK, S issued | waitP->gotP->gotV->PV issued]  softmax[waitS->S loaded->exp done->P arrived]")
for j in range(min(n, 24)):
    r = ch[j] - t0
    print(f"{j:2d}: K {r[8]:7d} {r[9]:7d} | P {r[10]:7d} {r[11]:7d} {r[12]:7d} {r[13]:7d} | sm {r[0]:7d} {r[1]:7d} {r[2]:7d} {r[3]:7d}")
v = ch[2:n - 1]
d = lambda a, b: float(np.mean(v[:, b] - v[:, a]))
print(f"means: softmax waitS {d(0,1):.0f} exp {d(1,2):.0f} store+arrive {d(2,3):.0f}; "
      f"issuer waitK {d(8,9):.0f} waitP {d(10,11):.0f} waitV {d(11,12):.0f} PVissue {d(12,13):.0f}")
print(f"chunk period (S issue) {float(np.mean(np.diff(ch[1:n, 9]))):.0f}")
nt = int((tl[:, 0] > 0).sum())
for it in range(min(nt, 6)):
    r = tl[it] - tl[it, 0]
    print(f"tile {it}: qempty {0} qfull(r0,r1) {r[6]} {r[7]}  sm end (g0,g1) {r[2]} {r[3]}  o_full (g0,g1) {r[4]} {r[5]}")
if nt > 2:
    print("tile period", float(np.mean(np.diff(tl[1:nt, 0]))))

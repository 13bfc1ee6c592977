"""Summarise a cached pass-0 timeline (FGA_CB_TRACE build, FGA_CB_TRACE_FILE=<file>): python scripts/cb_trace_report.py <file>"""
import numpy as np, sys
t = np.array([[int(x) for x in l.split()] for l in open(sys.argv[1]) if l.strip()], dtype=np.int64)
# slots: 0 prod before k_empty wait, 1 after; 2 mma before k_full, 3 after k_full, 4 after s_empty; 5 epi before s_full, 6 after s_full, 7 after compute
r = np.arange(16, 250)
def d(a, b): return (t[r, b] - t[r, a])
print("chunks with data", (t[:, 2] > 0).sum())
print("period (MMA issue, slot 4)", np.diff(t[r, 4]).mean(), " epilogue period (slot 6)", np.diff(t[r, 6]).mean())
print("producer wait k_empty", d(0, 1).mean())
print("issuer wait k_full", d(2, 3).mean(), " wait s_empty", d(3, 4).mean())
print("epilogue wait s_full", d(5, 6).mean(), " compute", d(6, 7).mean(), " 7->next 5", (t[r + 1, 5] - t[r, 7]).mean())
print("lead: s_full done minus issue", (t[r, 6] - t[r, 4]).mean())

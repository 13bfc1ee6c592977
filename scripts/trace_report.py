import numpy as np
t = np.loadtxt('gpurun_out/trace.txt', dtype=np.int64)
r = slice(5, 60)
print("period", np.diff(t[r, 5]).mean())
print(" mma: waitK", (t[r, 9] - t[r, 8]).mean(), "fence", (t[r, 13] - t[r, 9]).mean(), "S issue+commit", (t[r, 14] - t[r, 13]).mean())
print(" mma: waitP", (t[r, 11] - t[r, 10]).mean(), "PV(wait V+fence+issue+commit)", (t[r, 12] - t[r, 11]).mean())
print(" softmax: waitS", (t[r, 1] - t[r, 0]).mean(), "ld", (t[r, 2] - t[r, 1]).mean(), "max", (t[r, 3] - t[r, 2]).mean(),
      "exp", (t[r, 4] - t[r, 3]).mean(), "st", (t[r, 5] - t[r, 4]).mean())

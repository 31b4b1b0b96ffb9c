"""Summarise a GP_DEBUG_DUMP file by run phase (dev helper)."""
import sys
import numpy as np
a = np.loadtxt(sys.argv[1], dtype=np.float64)
n = len(a)
new, wmax, wavg = a[:, 5], a[:, 6], a[:, 7]
cmax, cavg = (a[:, 12], a[:, 13]) if a.shape[1] > 13 else (wmax, wavg)
r0, r1, r2, r3 = a[:, 1], a[:, 2], a[:, 3], a[:, 4]
nxt = np.r_[r0[1:] - r3[:-1], np.nan]
for lo, hi in [(0, n // 20), (n // 20, n // 10), (n // 10, n // 4), (n // 4, n // 2), (n // 2, 3 * n // 4), (3 * n // 4, n)]:
    sl = slice(lo, hi)
    m = lambda x: np.nanmedian(x[sl]) / 1e3
    print(f"{lo:6d}-{hi:6d} warp max {m(wmax):6.2f} avg {m(wavg):6.2f} | cta max {m(cmax):6.2f} avg {m(cavg):6.2f}"
          f" | fill+bar1 {m(r2 - r0):6.2f} sel {m(r3 - r2):5.2f} bar2 {m(nxt):5.2f} | new {new[sl].mean():.0f}")
tot = (r2 - r0).sum() / 1e6
print(f"sum fill+bar1 {tot:.1f} ms, sel {(r3 - r2).sum() / 1e6:.1f} ms, bar2 {np.nansum(nxt[nxt < 1e5]) / 1e6:.1f} ms")

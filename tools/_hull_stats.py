"""Pass-2 / pass-3 hull sizes on the bench scene (tuning aid)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O
o = np.fromfile(sys.argv[1], np.uint8).reshape(512, 512, 512)
rng = np.random.default_rng(0)
occ_sl = np.nonzero(o.any(axis=(1, 2)))[0]

def hull_size(rows, F):
    st = []
    for y, f in zip(rows, F):
        while len(st) >= 2:
            (ya, fa), (yb, fb) = st[-2], st[-1]
            if (fb - fa) * (y - yb) >= (f - fb) * (yb - ya):
                st.pop()
            else:
                break
        st.append((y, f))
    return len(st)

sizes = []
for _ in range(3000):
    i = int(rng.choice(occ_sl)); k = int(rng.integers(0, 512))
    sl = o[i]
    # 1D nearest site along k for each line j
    rows, F = [], []
    for j in range(512):
        ks = np.nonzero(sl[j])[0]
        if ks.size == 0:
            continue
        z = ks[np.argmin(np.abs(ks - k))]
        rows.append(j); F.append((k - int(z)) ** 2 + j * j)
    sizes.append(hull_size(rows, F))
sizes = np.array(sizes)
print("pass-2 hull size: mean %.1f median %d p90 %d p99 %d max %d; frac > 55: %.3f" % (
    sizes.mean(), np.median(sizes), np.percentile(sizes, 90), np.percentile(sizes, 99), sizes.max(), (sizes > 55).mean()))

import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(148, 64, 8).astype(np.int64)
names = ["tma_issue", "qk_issue", "pv_issue", "sm_sfull", "sm_pdone"]
for c in (0, 1, 50, 147):
    rows = t[c]
    base = rows[0, 0] if rows[0, 0] else rows[rows[:, 1] > 0][0, 1]
    print(f"CTA {c}:")
    for it in range(min(12, 64)):
        if rows[it, 1] == 0 and rows[it, 0] == 0:
            break
        print("   it", it, " ".join(f"{names[k]}={(rows[it, k]-base)/1e3 if rows[it,k] else -1:8.2f}" for k in range(5)))

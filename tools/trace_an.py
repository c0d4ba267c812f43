"""Print one K2 CTA's tile timeline from a kbench --dump trace (diagnostics)."""
import sys
import numpy as np
t = np.load(sys.argv[1]).astype(np.float64)
work = np.load(sys.argv[1].replace(".npy", "_work.npy"))
off = np.load(sys.argv[1].replace(".npy", "_ctaoff.npy"))
ctas = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 70]
R = lambda role: t[:, role * 256:(role + 1) * 256]
for c in ctas:
    c0 = t[c, 6 * 256 + 1]
    items = work[off[c]:off[c + 1]]
    print(f"CTA {c}: items (req, head, n_tok, keys, tiles):",
          [(int(w[0]), int(w[1]), int(w[3]), int(w[5] - w[4]), int((w[5] - w[4] + 63) // 64)) for w in items])
    n = int(sum((w[5] - w[4] + 63) // 64 for w in items))
    cols = [(0, "Ktop"), (4, "Kfree"), (5, "Kiss"), (10, "Vfree"), (11, "Viss"), (12, "mS"), (1, "S"),
            (8, "mPV"), (9, "Vland"), (7, "PV")]
    print("tile " + " ".join(f"{nm:>6s}" for _, nm in cols))
    for i in range(min(n, 256)):
        row = [(t[c, r * 256 + i] - c0) / 1e3 for r, _ in cols]
        print(f"{i:4d} " + " ".join(f"{v:6.2f}" for v in row))
    print("wg0 softmax (Sready, Pdone):", [((t[c, 2 * 256 + i] - c0) / 1e3, (t[c, 3 * 256 + i] - c0) / 1e3)
                                           for i in range((n + 1) // 2)])
    print("producer done / CTA done (kcycles):", (t[c, 6 * 256 + 2] - c0) / 1e3, (t[c, 6 * 256 + 3] - c0) / 1e3)
    nit = len(items)
    print("metadata staged (kcyc):", [round((t[c, 6 * 256 + 5 + i] - c0) / 1e3, 2) for i in range(nit)])
    for nm, r in (("epi entry", 13), ("epi O full", 14), ("epi O freed", 15)):
        print(f"{nm:12s}", [round((t[c, r * 256 + i] - c0) / 1e3, 2) for i in range(nit)])
    if t[c, 6 * 256 + 250] > 0:
        print("append start / done (kcyc):", (t[c, 6 * 256 + 250] - c0) / 1e3, (t[c, 6 * 256 + 251] - c0) / 1e3)

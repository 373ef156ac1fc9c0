"""Compare two polish_ab.py dumps: verdict / alive differences and ||delta|| agreement."""
import sys

import numpy as np


def main(fa, fb):
    a, b = np.load(fa), np.load(fb)
    ka = a["edge"].astype(np.int64) * 64 + a["obstacle"]
    kb = b["edge"].astype(np.int64) * 64 + b["obstacle"]
    ia, ib = np.argsort(ka), np.argsort(kb)
    assert np.array_equal(ka[ia], kb[ib])
    da, db, st = a["delta"][ia], b["delta"][ib], a["status"][ia]
    rel = np.abs(da - db) / np.maximum(np.abs(da), 1e-300)
    va, vb = (st == 0) & (da > 1e-7), (st == 0) & (db > 1e-7)
    sel = (st == 0) & (da > 1e-12)
    print(f"n {da.size} verdict diffs {int((va != vb).sum())} alive diffs {int((a['alive'] != b['alive']).sum())} "
          f"max rel ||delta|| diff {float(rel[sel].max()):.3e} exact-equal {float((da == db).mean()):.4f}")


if __name__ == "__main__":
    main(*sys.argv[1:])

"""Debug helper: find the shortest prefix of a stream where the GPU engine
and the CPU oracle disagree (run on the GPU box)."""
import sys
import numpy as np

sys.path.insert(0, ".")
from oracle.piecy_oracle import OracleEngine  # noqa: E402
from paper_1502_04265_b200 import BicoEngine  # noqa: E402


def same(X, W, d, m):
    g = BicoEngine(d, m)
    g.insert_block(X, W)
    o = OracleEngine(d, m)
    o.insert_block(X, W)
    lv, w, s, q, r = o.features()
    f = g.features()
    if len(f) != len(w):
        return False
    for i, (L, cf) in enumerate(f):
        if L != lv[i] or cf.weight != w[i] or not np.array_equal(cf.reference, r[i]) or not np.array_equal(cf.linear_sum, s[i]):
            return False
    return True


def main():
    seed = int(sys.argv[1]) if len(sys.argv) > 1 else 42
    rng = np.random.default_rng(seed)
    X = rng.normal(scale=4.0, size=(2000, 5))
    W = rng.integers(1, 9, size=2000)
    lo, hi = 1, 2000
    if same(X, W, 5, 25):
        print("no mismatch")
        return
    while lo < hi:
        mid = (lo + hi) // 2
        if same(X[:mid], W[:mid], 5, 25):
            lo = mid + 1
        else:
            hi = mid
    n = lo
    print("first mismatch at prefix", n, "item", n - 1, "w", W[n - 1])
    g = BicoEngine(5, 25); g.insert_block(X[:n], W[:n])
    o = OracleEngine(5, 25); o.insert_block(X[:n], W[:n])
    print("T", g.threshold, o.threshold, "F", g.num_features, o.num_features)
    lv, w, s, q, r = o.features()
    for i, (L, cf) in enumerate(g.features()):
        print(i, L, cf.weight, "|", lv[i] if i < len(w) else None, w[i] if i < len(w) else None,
              np.array_equal(cf.reference, r[i]) if i < len(w) else None)
    g2 = BicoEngine(5, 25); g2.insert_block(X[:n - 1], W[:n - 1])
    print("before item: ", [(L, cf.weight) for L, cf in g2.features()])
    print("x", X[n - 1])


if __name__ == "__main__":
    main()

"""Search for DRO inputs whose largest bucket attains the tight form of Lemma 1's count,
s*x + (p-1)(x-1) with x = ceil(ceil(n/p)/s), s = r p (reading Q10 of DESIGN.md, from the proof
at PAPER.md:430-476), and store them as tests/golden/dro_tight_instances.json.

Calls only oracle/ (test infrastructure): oracle.dro_sort gives the bucket counts, and a
hill-climb over the keys (single-key mutations, keep if the largest bucket does not shrink)
maximises the largest bucket.  The stored value is the oracle's; tests/test_oracle_pins.py pins
it with an independent brute-force re-derivation of Algorithm 1's split.

    python tools/gen_tight_instance.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def climb(n, p, r, seed, iters=20000, K=None):
    rng = np.random.default_rng(seed)
    K = K or n
    x = rng.integers(0, K, n).astype(np.int32)
    best = int(oracle.dro_sort(x, p, r).counts.max())
    tb = oracle.tight_bound(n, p, r)
    for _ in range(iters):
        if best >= tb:
            break
        y = x.copy()
        for _ in range(int(rng.integers(1, 3))):
            y[int(rng.integers(n))] = int(rng.integers(0, K))
        v = int(oracle.dro_sort(y, p, r).counts.max())
        if v >= best:
            x, best = y, v
    return x, best, tb


def main():
    oracle.build()
    found = []
    for (n, p, r) in [(12, 2, 1), (18, 3, 1), (20, 2, 2), (27, 3, 1), (36, 3, 2), (40, 4, 1), (50, 5, 1)]:
        for seed in range(40):
            x, best, tb = climb(n, p, r, seed)
            if best == tb:
                found.append({"n": n, "p": p, "r": r, "keys": [int(v) for v in x], "max_bucket": best,
                              "tight_bound": tb, "lemma1_bound": oracle.lemma1_bound(n, p, r),
                              "search_seed": seed})
                print(f"n={n} p={p} r={r}: max bucket {best} = tight bound (seed {seed})", flush=True)
                break
        else:
            print(f"n={n} p={p} r={r}: not attained (best {best} < {tb})", flush=True)
    out = {"source": "tools/gen_tight_instance.py (hill-climb over oracle.dro_sort, balanced positions)",
           "cite": "Lemma 1 proof, PAPER.md:430-476: a bucket holds at most s*x keys of the sample segments "
                   "around its splitter plus x-1 keys of every other sequence (reading Q10 of DESIGN.md)",
           "instances": found}
    path = os.path.join(ROOT, "tests", "golden", "dro_tight_instances.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, len(found), "instances")


if __name__ == "__main__":
    main()

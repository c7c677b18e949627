"""Full-size goldens from the REFERENCE ITSELF (oracle/_ref/libref.so), stored
as SHA-256 digests so they stay small: tests/golden/large.npz.

* xoshiro256**: the first 1e6 draws of Rng(derive_seed(1, 1))
* global_reset on n = 1e6 (rho 0.5, 0.8): chosen set + next draw
* C3 = ER(1e5, p=1e-4, seed 1): the CSR, MIS-QUBO steps t = 1, 10 (x, v)
* one_two_swap on C3 from greedy_maximalize(g, {}); one_two_flip on
  BA(1e5, 5, seed 2) from random sides

Run here (where /root/reference exists):  python tests/golden/make_large_golden.py
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "large.npz")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    oracle.build(ref=True)
    R = oracle.load("ref")
    assert R.name == "reference"
    z = {}
    r = R.rng(R.derive_seed(1, 1))
    z["stream_1e6_sha"] = np.array(sha(np.array([r.next_u64() for _ in range(1_000_000)],
                                                np.uint64)))
    for rho in (0.5, 0.8):
        r = R.rng(R.derive_seed(1_000_000, int(rho * 10)))
        _, chosen = R.global_reset(np.ones(1_000_000), rho, r)
        z[f"reset_1e6_{rho}_sha"] = np.array(sha(chosen))
        z[f"reset_1e6_{rho}_next"] = np.array([r.next_u64()], np.uint64)
    g = R.generate_er(100_000, 1e-4, 1)
    off, nbr = g.csr()
    z["c3_csr_sha"] = np.array(sha(off, nbr))
    x0 = np.random.default_rng(33).uniform(0.0, 1.0, g.n)
    x, v = x0.copy(), np.zeros(g.n)
    for t in range(1, 11):
        x, v = R.step(g, oracle.MIS_QUBO, 2.0, x, v, 0.8, 0.3)
        if t in (1, 10):
            z[f"c3_x{t}_sha"] = np.array(sha(x))
            z[f"c3_v{t}_sha"] = np.array(sha(v))
    ind, _ = R.greedy_maximalize(g, np.zeros(g.n, np.uint8))
    z["c3_greedy_sha"] = np.array(sha(ind))
    ind2, size = R.one_two_swap(g, ind)
    z["c3_swap_sha"] = np.array(sha(ind2))
    z["c3_swap_size"] = np.array([size], np.int64)
    gb = R.generate_ba(100_000, 5, 2)
    side = np.random.default_rng(1).integers(0, 2, gb.n).astype(np.uint8)
    s3, gain = R.one_two_flip(gb, side)
    z["ba1e5_onetwo_sha"] = np.array(sha(s3))
    z["ba1e5_onetwo_gain"] = np.array([gain], np.int64)
    np.savez_compressed(OUT, **z)
    print("wrote", OUT, {k: (str(v)[:16] if v.dtype.kind == "U" else v.tolist()) for k, v in z.items()})


if __name__ == "__main__":
    main()

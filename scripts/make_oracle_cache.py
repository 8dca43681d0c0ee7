"""Write tests/golden/oracle_cache.npz: the CPU oracle's expected outputs at BASELINE.json's
full sizes, for the full-size GPU parity tests (tests/test_gpu_fullsize.py).

Calls ONLY oracle/ (the plain CPU oracle: literal Algorithm 2 per source, and
the plain largest-WCC labelling, Table 1) and graphgen/ (seeded inputs).  Nothing here
reads the CUDA path.  Re-run after any change to graphgen or the oracle:

    python scripts/make_oracle_cache.py          # ~5 min on 8 cores
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402
import oracle  # noqa: E402


def fingerprint(g):
    return np.array([g.n, g.m, int(g.col.astype(np.int64).sum()),
                     int((g.row_ptr[1:] * np.arange(1, g.n + 1, dtype=np.int64)).sum() & 0x7FFFFFFFFFFFFFFF)],
                    dtype=np.int64)


def main():
    out = {}
    t0 = time.time()
    # C5: every source of the largest WCC of Kronecker-18 (APSP, E11-E12)
    g = graphgen.config_graph("C5")
    verts, e_wcc = oracle.largest_wcc(g.n, g.row_ptr, g.col)
    out["c5_fp"] = fingerprint(g)
    out["c5_verts"] = verts.astype(np.int64)
    out["c5_e_wcc"] = np.array([e_wcc], np.int64)
    out["c5_records"] = oracle.records(g.n, g.row_ptr, g.col, verts)
    print(f"C5: {len(verts)} records, {time.time() - t0:.0f} s", flush=True)
    # C2 / C4: the 64 bench sources of rank 0 (seed 1), one record per distance row
    for cfg in ("C2", "C4"):
        t = time.time()
        g = graphgen.config_graph(cfg)
        srcs = g.sample_sources(64, seed=1).astype(np.int64)
        out[f"{cfg.lower()}_fp"] = fingerprint(g)
        out[f"{cfg.lower()}_sources"] = srcs
        out[f"{cfg.lower()}_records"] = oracle.records(g.n, g.row_ptr, g.col, srcs)
        print(f"{cfg}: 64 records, {time.time() - t:.0f} s", flush=True)
        del g
    path = os.path.join(ROOT, "tests", "golden", "oracle_cache.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()

"""Generate the reference golden fixtures (run in the dev container only).

For every BASELINE.json configuration (and a few small shapes) this runs the
UNMODIFIED reference, compiled from /root/reference by `make ref` into
oracle/_ref, on the synthetic matrix produced by this repo's generator, and
records hashes of everything the hot path's parity depends on:

  * the ordering / range partition / PᵀAP / IC(k) pattern (reference analyze,
    pipeline.hpp:35-55) -- pins this repo's host analysis;
  * the block structure (build_block_matrix, block_layout.hpp:98-181) and the
    task DAG (export_task_dag, factorize.hpp:260-302) -- pins the flattener;
  * the factor values of factor_serial (factorize.hpp:94-130) -- pins the
    plain-C oracle, which the GPU tests then compare against;
  * the pattern-restricted residual of that factor.

Hash: h = (h ^ bits(x)) * 1099511628211, h0 = 1469598103934665603, over 64-bit
words; ints are sign-extended.

    python tests/golden/make_golden.py            # writes tests/golden/golden.json
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_1601_05871_b200 as T  # noqa: E402
from checkers import Oracle, Reference  # noqa: E402

# name: (generator kind, p0, p1, seed, level, leaf_size)
CASES = {
    "c1": ("grid2d", 100, 100, 0, 0, 64),
    "c2": ("lap7", 64, 0, 0, 1, 64),
    "c3": ("stencil27", 48, 0, 1, 2, 64),
    "c4": ("elasticity", 40, 0, 1, 0, 64),
    "c5_m0": ("diffusion", 32, 1000, 1, 1, 64),
    "c5_m63": ("diffusion", 32, 1000, 64, 1, 64),
    "c6": ("lap7", 128, 0, 0, 1, 64),
    "s27_16_k2": ("stencil27", 16, 0, 1, 2, 64),   # SURVEY §8(c) survey-probe hash
    "grid20_k2_leaf4": ("grid2d", 20, 20, 0, 2, 4),
    "rand_spd_200": ("random_spd", 200, 20000, 7, 1, 8),
    "elast6_k1": ("elasticity", 6, 0, 3, 1, 16),
}


# The reference's own test generators (tests/support/test_matrices.hpp) against
# which this repo's grid2d / path / random_spd are pinned: (reference kind,
# this repo's kind, p0, p1, seed)
REF_GENERATORS = {
    "grid_100x100": ("grid", "grid2d", 100, 100, 0),      # BASELINE.json configs[0]
    "grid_20x20": ("grid", "grid2d", 20, 20, 0),
    "grid_7x13": ("grid", "grid2d", 7, 13, 0),
    "path_1000": ("path", "path", 1000, 0, 0),
    "random_spd_200_s7": ("random_spd", "random_spd", 200, 20000, 7),
    "random_spd_60_s1": ("random_spd", "random_spd", 60, 150000, 1),
    "random_spd_333_s42": ("random_spd", "random_spd", 333, 8000, 42),
}


def reference_generators(golden):
    """Hashes of the matrices the reference's test generators produce."""
    O, R = Oracle(), Reference()
    out = {}
    for name, (rkind, kind, p0, p1, seed) in REF_GENERATORS.items():
        ptr, col, val = R.test_matrix(rkind, p0, p1, seed)
        out[name] = {"reference_kind": rkind, "kind": kind, "args": [p0, p1, seed], "n": int(len(ptr) - 1),
                     "nnz": int(len(col)), "row_ptr": O.hash(ptr), "col_idx": O.hash(col), "values": O.hash(val)}
        print(f"reference generator {name}: n={out[name]['n']} nnz={out[name]['nnz']} values={out[name]['values']}")
    golden["reference_generators"] = out


def main(names):
    O, R = Oracle(), Reference()
    out_path = os.path.join(HERE, "golden.json")
    golden = json.load(open(out_path)) if os.path.exists(out_path) else {}
    reference_generators(golden)
    for name in names:
        kind, p0, p1, seed, level, leaf = CASES[name]
        t0 = time.time()
        a = T.generate(kind, p0, p1, seed)
        ra = R.analyze(a, level=level, leaf=leaf)
        u = T.CsrMatrix.from_arrays(a.nrows, ra["u_ptr"], ra["u_col"])
        ap = T.CsrMatrix.from_arrays(a.nrows, ra["a_ptr"], ra["a_col"], ra["a_val"])
        kinds, bi, bj, ef, et = R.export_dag(u, ra["bounds"])
        bp, bc = R.blocks(u, ra["bounds"])
        vals, st, secs, brow, bpiv = R.factor_serial(ap, u)
        rec = {
            "generator": [kind, p0, p1, seed], "level": level, "leaf_size": leaf,
            "n": a.nrows, "nnz_a": a.nnz(), "nnz_u": u.nnz(), "nranges": len(ra["bounds"]) - 1,
            "raw": {"row_ptr": O.hash(a.row_ptr), "col_idx": O.hash(a.col_idx), "values": O.hash(a.values)},
            "perm": O.hash(ra["perm"]), "bounds": O.hash(ra["bounds"]),
            "a_permuted": {"row_ptr": O.hash(ap.row_ptr), "col_idx": O.hash(ap.col_idx),
                           "values": O.hash(ap.values)},
            "pattern": {"row_ptr": O.hash(u.row_ptr), "col_idx": O.hash(u.col_idx)},
            "blocks": {"nblocks": int(len(bc)), "brow_ptr": O.hash(bp), "bcol_idx": O.hash(bc)},
            "dag": {"nodes": int(len(kinds)), "edges": int(len(ef)),
                    "tasks": [int((kinds == k).sum()) for k in range(4)],
                    "kind": O.hash(kinds), "block_row": O.hash(bi), "block_col": O.hash(bj),
                    "edge_from": O.hash(ef), "edge_to": O.hash(et)},
            "factor_status": int(st),
            "factor_values": O.hash(vals) if st == 0 else None,
            "residual": float(O.residual(ap, u, vals)) if st == 0 else None,
            "serial_seconds_devbox": secs,
        }
        golden[name] = rec
        print(f"{name}: n={rec['n']} nnz_u={rec['nnz_u']} tasks={rec['dag']['nodes']} "
              f"values={rec['factor_values']} ({time.time() - t0:.1f}s)", flush=True)
    json.dump(golden, open(out_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))

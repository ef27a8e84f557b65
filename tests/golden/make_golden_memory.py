"""Golden fixtures for the memory-pressure refine paths (refine.cpp:160-183,
343-350), minted from the UNMODIFIED reference (oracle/_ref) on the local
graphs of distributed.npz:

  skip_tree_phase, max_concat_bytes = 1 (forces the skip) and = 1 GiB (no
  skip) at P = 4 and P = 8, and M = 4 at P = 8 with and without
  double_buffer (three flat steps, the prefetch path).

    python tests/golden/make_golden_memory.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.bindings import Ref  # noqa: E402

CASES = {
    # name: (P, M, skip_tree, max_concat_bytes, double_buffer, beam, entries)
    "p4_skip": (4, 2, True, 0, False, 64, 16),
    "p4_concat1": (4, 2, False, 1, False, 64, 16),
    "p4_concat1g": (4, 2, False, 1 << 30, False, 64, 16),
    "p8_skip": (8, 2, True, 0, False, 128, 96),
    "p8_concat1": (8, 2, False, 1, False, 128, 96),
    "p8_m4": (8, 4, False, 0, False, 64, 16),
    "p8_m4_db": (8, 4, False, 0, True, 64, 16),
}


def main():
    R = Ref()
    g = np.load(os.path.join(HERE, "distributed.npz"))
    x = g["x"]
    out = {}
    for name, (P, M, skip, mcb, db, beam, ent) in CASES.items():
        cfg = R.refine_config(P, M, 16, nn_seed=2, search_seed=2, seed=2, beam_width=beam,
                              num_entry_points=ent, skip_tree=skip, max_concat_bytes=mcb,
                              double_buffer=db)
        li, ld = g[f"local{P}_ids"], g[f"local{P}_d"]
        ri, rd = R.refine_from_local(x, cfg, li, ld, 0)
        out[name + "_ids"], out[name + "_d"] = ri, rd
        print(name, "done", flush=True)
    np.savez_compressed(os.path.join(HERE, "memory_paths.npz"), **out)


if __name__ == "__main__":
    main()

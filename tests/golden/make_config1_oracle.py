"""Oracle scores of BASELINE config 1 (the 1,024-pose slice bench.py's parity
block and tests/test_gpu_config1.py score): pocket 1,000 atoms (seed 0),
ligands U{16..64} (seed 1), FusionModel(seed=0), coherent fusion.

    python tests/golden/make_config1_oracle.py     # ~1 min on 8 cores

The oracle (oracle/fusion_oracle.py) is itself pinned to the unmodified
reference's goldens (tests/test_oracle_golden.py); this fixture only saves
the GPU tests from re-running 1,024 float64 poses on the GPU box.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    scores, rate = bench.cpu_oracle_pool(1024, os.cpu_count() or 1)
    out = os.path.join(ROOT, "tests", "golden", "config1_oracle.npz")
    np.savez_compressed(out, scores=scores)
    print(f"wrote {out}: {len(scores)} scores ({rate:.1f} poses/s)")


if __name__ == "__main__":
    main()

"""Generate SSHC/SSHS fixture files with the REFERENCE's own writer.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_io_fixtures.py

tests/test_io.py checks that paper_1110_6298_b200.io reads these files to the
same values and writes byte-identical files (pkg/src/torusht/io.py).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import torusht as ref  # noqa: E402
from torusht import io as ref_io  # noqa: E402

from oracle.mw_oracle import gaussian_coeffs  # noqa: E402

v = gaussian_coeffs(6, -2, 9)
ref_io.save_coeffs(os.path.join(HERE, "io_L6_s-2.sshc"), ref.HarmonicCoeffs(6, -2, v))
sig = ref.inverse(ref.HarmonicCoeffs(6, -2, v)).samples
ref_io.save_signal(os.path.join(HERE, "io_L6_s-2.sshs"), np.asarray(sig), -2)
ref_io.save_coeffs(os.path.join(HERE, "io_L3_s0_gl.sshc"),
                   ref.HarmonicCoeffs(3, 0, gaussian_coeffs(3, 0, 1)), grid="gl")
print("wrote", sorted(f for f in os.listdir(HERE) if f.startswith("io_")))

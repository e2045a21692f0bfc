"""pytest plugin: register this repo's `cuda_kernels` in the reference's backend registry
 before the reference's own test suite imports anything.

    TRITPACK_BACKEND=cuda python -m pytest -p ref_cuda_plugin baseline/_ref/tritpack_tests  (tests/ on PYTHONPATH)

(scripts/run_reference_suite.sh); with TRITPACK_BACKEND=cuda every reference call that uses
the default backend runs on the B200 kernels.
"""

import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(_ROOT, "baseline", "_ref"))
sys.path.insert(0, _ROOT)

from tritpack import backend  # noqa: E402

from paper_2506_23025_b200 import cuda_kernels  # noqa: E402

backend._BY_NAME["cuda"] = cuda_kernels

"""``piecy`` resolving to the B200 drop-in (paper_1502_04265_b200), so the
reference's own test suite (pkg/tests) runs against it: hot-path modules map
to the drop-in, the out-of-scope linalg helpers come from the unmodified
reference (``_ref``).  Test scaffolding only -- see tools/run_ref_tests.sh."""

import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if _REPO not in sys.path:
    sys.path.insert(0, _REPO)

from paper_1502_04265_b200 import *  # noqa: E402,F401,F403
from paper_1502_04265_b200 import __version__  # noqa: E402,F401

from .linalg import exact_truncated_svd, reconstruction_error, spectrum  # noqa: E402,F401

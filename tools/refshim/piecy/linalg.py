"""piecy.linalg -> paper_1502_04265_b200.linalg; exact_truncated_svd,
spectrum and reconstruction_error (out of scope: test oracles) from the
unmodified reference."""
import sys

from paper_1502_04265_b200 import linalg as _m
from paper_1502_04265_b200.linalg import *  # noqa: F401,F403

from ._ref import load as _load

_self = sys.modules[__name__]
for _k, _v in vars(_m).items():
    if not _k.startswith("__") and not hasattr(_self, _k):
        setattr(_self, _k, _v)
_R = _load()
exact_truncated_svd = _R.linalg.exact_truncated_svd
spectrum = _R.linalg.spectrum
reconstruction_error = _R.linalg.reconstruction_error

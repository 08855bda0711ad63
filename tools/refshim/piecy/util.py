"""piecy.util -> paper_1502_04265_b200.util (drop-in under test)."""
import sys

from paper_1502_04265_b200 import util as _m
from paper_1502_04265_b200.util import *  # noqa: F401,F403

# the module's public names, underscored helpers included, as the reference's tests see them
_self = sys.modules[__name__]
for _k, _v in vars(_m).items():
    if not _k.startswith("__") and not hasattr(_self, _k):
        setattr(_self, _k, _v)

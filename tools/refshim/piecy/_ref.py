"""The unmodified reference package under the alias ``_piecy_ref``, for the
out-of-scope helpers the drop-in does not rebuild (exact SVD, spectrum,
reconstruction error: test oracles and paper figures).
It is the pip --target install in baseline/_ref (git-ignored, travels to the
GPU box); /root/reference itself is never read."""

import importlib.util
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def load():
    if "_piecy_ref" in sys.modules:
        return sys.modules["_piecy_ref"]
    root = os.environ.get("PIECY_REF_DIR") or os.path.join(_ROOT, "baseline", "_ref", "piecy")
    spec = importlib.util.spec_from_file_location("_piecy_ref", os.path.join(root, "__init__.py"),
                                                  submodule_search_locations=[root])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_piecy_ref"] = mod
    spec.loader.exec_module(mod)
    return mod

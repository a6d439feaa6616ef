"""Tools only: point the binding at a measurement build (VARIANT_LIB=path/to/libbmc_b200.so)
before anything loads the library.  The product package never reads this variable."""
import os
from pathlib import Path


def use_variant_from_env():
    path = os.environ.get("VARIANT_LIB")
    if not path:
        return None
    from paper_2508_05990_b200 import _native as N
    N._LIB_PATH = Path(path).resolve()
    N.load(build_if_missing=False)
    return N._LIB_PATH

"""Import the UNMODIFIED reference package (/root/reference) with its compiled
core taken from oracle/_ref (built by oracle/build_ref.sh).  Used only by the
golden-fixture generator in this directory; never at test time (the reference
tree does not exist on the GPU box)."""
import importlib.util
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_SRC = os.environ.get("REF_ROOT", "/root/reference") + "/pkg/src"


def import_reference():
    sys.path.insert(0, REPO)
    from oracle import oracle as O

    path = O.reference_path()
    if path is None:
        raise RuntimeError("oracle/_ref not built: run `make -C oracle`")
    spec = importlib.util.spec_from_file_location("adascale._kernels", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    sys.modules["adascale._kernels"] = mod
    sys.path.insert(0, REF_SRC)
    import adascale

    assert adascale.active_core() == "compiled", adascale.active_core()
    return adascale

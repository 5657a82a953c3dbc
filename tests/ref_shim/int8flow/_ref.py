"""The unmodified reference package, loaded from ``baseline/_ref`` under a private
name (``_int8flow_ref``) so it does not collide with this shim's ``int8flow``."""

import importlib.util
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
REF_DIR = os.environ.get("JF_REF_PKG", os.path.join(_ROOT, "baseline", "_ref", "int8flow"))


def _load():
    name = "_int8flow_ref"
    if name in sys.modules:
        return sys.modules[name]
    init = os.path.join(REF_DIR, "__init__.py")
    if not os.path.exists(init):
        raise ImportError(f"reference package not installed at {REF_DIR} (tools/install_reference.sh)")
    spec = importlib.util.spec_from_file_location(name, init, submodule_search_locations=[REF_DIR])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


ref = _load()
qtensor = sys.modules["_int8flow_ref.qtensor"]
qgemm = sys.modules["_int8flow_ref.qgemm"]
qnonlinear = sys.modules["_int8flow_ref.qnonlinear"]
qlayers = sys.modules["_int8flow_ref.qlayers"]

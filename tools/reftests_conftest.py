"""conftest for running the REFERENCE's own test suite (pkg/tests of gks3d)
against this package: `gks3d.*` is aliased to paper_2304_09485_b200.*
(tools/run_reference_tests.sh copies the tests next to this file in a
scratch directory; nothing of the reference is committed).

Names a reference test imports that the drop-in does not provide (the
reference's internal helpers: host ghost-state functions, reconstruction
classes, the CLI, report plots) resolve to stubs raising
NotImplementedError, so each test module still collects and the outcome is
reported per test."""
import importlib
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ALIAS = {
    "gks3d": ["paper_2304_09485_b200"],
    "gks3d.flux": ["paper_2304_09485_b200.flux"],
    "gks3d.kinetic": ["paper_2304_09485_b200.kinetic"],
    "gks3d.stepping": ["paper_2304_09485_b200.stepping"],
    "gks3d.boundary": ["paper_2304_09485_b200.boundary"],
    "gks3d.jacobian": ["paper_2304_09485_b200.jacobian"],
    "gks3d.krylov": ["paper_2304_09485_b200.krylov"],
    "gks3d.config": ["paper_2304_09485_b200.config"],
    "gks3d.driver": ["paper_2304_09485_b200.driver"],
    "gks3d.output": ["paper_2304_09485_b200.output"],
    "gks3d.hweno": ["paper_2304_09485_b200.hweno"],
    "gks3d.mesh": ["paper_2304_09485_b200.mesh", "paper_2304_09485_b200.stencils"],
    "gks3d.mesh.geometry": ["paper_2304_09485_b200.mesh"],
    "gks3d.mesh.boxgen": ["paper_2304_09485_b200.mesh"],
    "gks3d.mesh.fileio": ["paper_2304_09485_b200.mesh"],
    "gks3d.mesh.stencils": ["paper_2304_09485_b200.stencils"],
    "gks3d.recon": ["paper_2304_09485_b200.recon"],
    "gks3d.cli": [],
    "gks3d.report": [],
}


def _stub(modname, name):
    def f(*a, **k):
        raise NotImplementedError(f"{modname}.{name} is not part of the drop-in")
    f.__name__ = name
    return f


def _alias(name, targets):
    m = types.ModuleType(name)
    m.__path__ = []  # importable as a package
    for t in targets:
        m.__dict__.update({k: v for k, v in vars(importlib.import_module(t)).items() if not k.startswith("__")})
    def getattr_(attr, _n=name):
        if attr.startswith("__"):
            raise AttributeError(attr)
        return _stub(_n, attr)

    m.__getattr__ = getattr_
    return m


for _name, _targets in ALIAS.items():
    sys.modules[_name] = _alias(_name, _targets)
for _name in ALIAS:
    if "." in _name:
        parent, child = _name.rsplit(".", 1)
        setattr(sys.modules[parent], child, sys.modules[_name])

# the reference's oracle module (test support, copied beside the tests)
_here = Path(__file__).resolve().parent
if (_here / "gks3d_oracles.py").exists():
    spec = importlib.util.spec_from_file_location("gks3d.oracles", _here / "gks3d_oracles.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["gks3d.oracles"] = mod
    spec.loader.exec_module(mod)

"""Every `from <package module> import name` in the package, tools, tests
and bench -- including the lazy ones inside functions, which only run on a
GPU box or in multi-process mode -- names something that exists (a removed
helper must fail here, on CPU, not on the GPU box)."""

import ast
import importlib
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = "paper_2408_04307_b200"
FILES = sorted(list((ROOT / PKG).glob("*.py")) + list((ROOT / "tools").glob("*.py")) +
               list((ROOT / "tests").glob("test_*.py")) +
               [ROOT / "bench.py", ROOT / "__graft_entry__.py",
                ROOT / "examples" / "moe_training.py"])


def _imports(path: Path):
    tree = ast.parse(path.read_text())
    for node in ast.walk(tree):
        if isinstance(node, ast.ImportFrom) and node.module is not None:
            mod = node.module
            if node.level:  # relative import inside the package
                mod = f"{PKG}.{mod}" if mod else PKG
            if mod == PKG or mod.startswith(PKG + ".") or mod == "oracle" or \
                    mod.startswith("oracle."):
                yield mod, [a.name for a in node.names]


@pytest.mark.parametrize("path", FILES, ids=lambda p: str(p.relative_to(ROOT)))
def test_package_imports_resolve(path):
    for mod, names in _imports(path):
        m = importlib.import_module(mod)
        for n in names:
            if n == "*":
                continue
            if not hasattr(m, n):
                importlib.import_module(f"{mod}.{n}")  # a submodule


def test_product_never_imports_the_oracle():
    """The oracle is test infrastructure: no module of the package (the
    product path) may import it, statically or lazily, and importing the
    package (with its native library) must not pull it in."""
    import subprocess
    import sys
    for path in sorted((ROOT / PKG).glob("*.py")):
        tree = ast.parse(path.read_text())
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom) and node.module and node.level == 0:
                names = [node.module]
            for n in names:
                assert n != "oracle" and not n.startswith("oracle."), (path.name, n)
        assert "pec_oracle" not in path.read_text(), path.name
    code = ("import sys, paper_2408_04307_b200 as p; from paper_2408_04307_b200 import device, "
            "snapshot, restore, store, staging; device.lib(); "
            "print(sorted(m for m in sys.modules if m == 'oracle' or m.startswith('oracle.')))")
    res = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert res.stdout.strip() == "[]", res.stdout

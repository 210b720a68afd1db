"""Static guard for the GPU-only code paths (CPU suite): every name a module
of the package loads is bound somewhere in that module (import, def, class,
assignment, argument) or is a builtin -- catches a renamed helper on a path
the CPU tests cannot execute."""

import ast
import builtins
import pathlib

import pytest

PKG = pathlib.Path(__file__).resolve().parents[1] / "paper_2101_08053_b200"


@pytest.mark.parametrize("path", sorted(PKG.glob("*.py")), ids=lambda p: p.name)
def test_no_unbound_names(path):
    tree = ast.parse(path.read_text())
    bound = set(dir(builtins)) | {"__file__", "__name__"}
    for n in ast.walk(tree):
        if isinstance(n, (ast.FunctionDef, ast.AsyncFunctionDef, ast.ClassDef)):
            bound.add(n.name)
        elif isinstance(n, ast.Import):
            bound.update((a.asname or a.name).split(".")[0] for a in n.names)
        elif isinstance(n, ast.ImportFrom):
            bound.update(a.asname or a.name for a in n.names)
        elif isinstance(n, ast.Name) and isinstance(n.ctx, (ast.Store, ast.Del)):
            bound.add(n.id)
        elif isinstance(n, ast.arg):
            bound.add(n.arg)
        elif isinstance(n, ast.ExceptHandler) and n.name:
            bound.add(n.name)
    used = {n.id for n in ast.walk(tree) if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Load)}
    assert not sorted(used - bound)

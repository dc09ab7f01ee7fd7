"""smoke() and bench.py's GPU arm cannot run in the CPU suite; this catches the cheapest way to
break them unseen — a name that is read but bound nowhere in the file (a half-applied edit)."""
import ast
import builtins
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def unbound_names(path: Path) -> list[str]:
    tree = ast.parse(path.read_text())
    bound = set(dir(builtins)) | {"__file__", "__name__"}
    for n in ast.walk(tree):
        if isinstance(n, (ast.Import, ast.ImportFrom)):
            bound.update((a.asname or a.name).split(".")[0] for a in n.names)
        elif isinstance(n, (ast.FunctionDef, ast.AsyncFunctionDef, ast.Lambda)):
            if not isinstance(n, ast.Lambda):
                bound.add(n.name)
            args = n.args
            bound.update(a.arg for a in args.args + args.kwonlyargs + args.posonlyargs)
            bound.update(a.arg for a in (args.vararg, args.kwarg) if a)
        elif isinstance(n, ast.ClassDef):
            bound.add(n.name)
        elif isinstance(n, ast.Name) and isinstance(n.ctx, (ast.Store, ast.Del)):
            bound.add(n.id)
        elif isinstance(n, ast.ExceptHandler) and n.name:
            bound.add(n.name)
    return [f"{path.name}:{n.lineno}: {n.id}" for n in ast.walk(tree)
            if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Load) and n.id not in bound]


@pytest.mark.parametrize("rel", ["__graft_entry__.py", "bench.py", "paper_2402_15281_b200/api.py",
                                 "paper_2402_15281_b200/abi.py", "paper_2402_15281_b200/parallel.py",
                                 "tests/parity_report.py"])
def test_no_name_is_read_but_never_bound(rel):
    assert unbound_names(ROOT / rel) == []

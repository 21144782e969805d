"""The product path never touches the oracle and fails loudly without its
native library (no CPU fallback)."""
import ast
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2510_00606_b200"


def test_package_never_imports_the_oracle():
    for py in PKG.rglob("*.py"):
        tree = ast.parse(py.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            else:
                continue
            assert not any(n.split(".")[0] == "oracle" for n in names), (py, names)
    import re
    for src in (PKG / "csrc").rglob("*"):
        if src.suffix in (".cpp", ".cu", ".cuh", ".h", ".hpp"):
            text = src.read_text()
            assert not re.search(r'#include\s+["<][^">]*oracle', text), src
            assert not re.search(r"\bew_oracle_\w+\s*\(", text), src  # citations are fine, calls are not


def test_missing_library_fails_loudly(tmp_path):
    clone = tmp_path / "paper_2510_00606_b200"
    shutil.copytree(PKG, clone, ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    code = ("import sys; sys.path.insert(0, %r)\n"
            "try:\n import paper_2510_00606_b200\nexcept ImportError as e:\n"
            " print('IMPORT_ERROR', e)\n" % str(tmp_path))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=300).stdout
    assert "IMPORT_ERROR" in out and "no fallback" in out

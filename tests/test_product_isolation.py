"""The product path never reaches the oracle (task contract):
no module of the package imports oracle/, no CUDA source includes anything
from it, and the binding raises instead of falling back when the library is
missing."""
import ast
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2504_17785_b200")


def _imports(path):
    tree = ast.parse(open(path).read(), path)
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            yield from (a.name for a in node.names)
        elif isinstance(node, ast.ImportFrom) and node.level == 0:
            yield node.module or ""


def test_package_does_not_import_oracle():
    for name in sorted(os.listdir(PKG)):
        if name.endswith(".py"):
            mods = list(_imports(os.path.join(PKG, name)))
            assert not any(m == "oracle" or m.startswith("oracle.") for m in mods), (name, mods)


def test_cuda_sources_do_not_include_oracle():
    csrc = os.path.join(PKG, "csrc")
    for name in sorted(os.listdir(csrc)):
        for line in open(os.path.join(csrc, name), errors="replace"):
            if re.match(r"\s*#\s*include", line):
                assert "oracle" not in line, (name, line)


def test_binding_fails_loudly_without_library(tmp_path):
    code = ("import os, sys; sys.path.insert(0, %r)\n"
            "from paper_2504_17785_b200 import silenzio\n"
            "try:\n    silenzio.load()\nexcept Exception as e:\n    print('raised', type(e).__name__)\n"
            "else:\n    print('loaded')\n") % ROOT
    env = dict(os.environ, SILENZIO_LIB=str(tmp_path / "missing.so"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert "raised" in out.stdout, out.stdout + out.stderr

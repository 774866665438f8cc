"""The product never routes through the oracle or a CPU fallback: no module
of the package imports oracle/ or numba, and the SpMV entry point reaches
the native library (checked without a GPU by source inspection)."""

import ast
import os

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_2307_06305_b200")


def _imports(path):
    tree = ast.parse(open(path).read())
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            for n in node.names:
                yield n.name
        elif isinstance(node, ast.ImportFrom):
            yield node.module or ""


def test_package_never_imports_oracle_or_cpu_backends():
    for name in os.listdir(PKG):
        if name.endswith(".py"):
            mods = set(_imports(os.path.join(PKG, name)))
            assert not any(m.split(".")[0] in ("oracle", "numba", "dacsr") for m in mods), name


def test_spmv_compute_goes_through_the_c_abi():
    src = open(os.path.join(PKG, "device.py")).read()
    assert "dacsr_spmv" in src
    tree = ast.parse(open(os.path.join(PKG, "spmv.py")).read())
    # no host arithmetic on the matrix in the operator: only validation and copies
    matmul = [n for n in ast.walk(tree) if isinstance(n, ast.BinOp) and isinstance(n.op, ast.MatMult)]
    calls = {n.func.attr for n in ast.walk(tree)
             if isinstance(n, ast.Call) and isinstance(n.func, ast.Attribute)}
    assert not matmul and not ({"dot", "matmul", "einsum"} & calls)

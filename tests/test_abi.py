"""The C-ABI drop-in boundary: libaqp.so is built for sm_100a, loads, exports
exactly the entry points include/aqp.h declares, and the ctypes mirrors of
its structs have the C layout.  No compute call is made (CPU-only test)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2602_23967_b200 import _native as nat
from paper_2602_23967_b200 import build

HEADER = os.path.join(ROOT, "include", "aqp.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aqp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return nat.load()


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (aqp_[a-z0-9_]+)", out))
    missing = [f for f in declared() if f not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(lib):
    assert sorted(nat.SIGNATURES) == declared()
    assert lib.aqp_abi_version() == nat.ABI_VERSION == 3


def test_library_is_sm100a():
    res = subprocess.run(["cuobjdump", "--list-elf", nat.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in res.stdout


def _c_layout():
    code = r'''
#include <stdio.h>
#include <stddef.h>
#include "aqp.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(aqp_problem_desc), sizeof(aqp_problem_info),
         sizeof(aqp_solver_params), sizeof(aqp_scalars), sizeof(aqp_check_result), sizeof(aqp_shard_desc),
         sizeof(aqp_setup_info));
  printf("%zu %zu %zu %zu %zu %zu\n", offsetof(aqp_problem_desc, con_hi), offsetof(aqp_check_result, xr_qd_inf),
         offsetof(aqp_scalars, have_avg_prev), offsetof(aqp_problem_desc, shard), offsetof(aqp_shard_desc, yw),
         offsetof(aqp_setup_info, diag_bound));
  return 0;
}'''
    exe = os.path.join(ROOT, "build", "abi_probe")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["gcc", "-x", "c", "-", "-I", os.path.join(ROOT, "include"), "-o", exe], input=code, text=True,
                   check=True)
    return [list(map(int, line.split())) for line in subprocess.run([exe], capture_output=True, text=True).stdout.splitlines()]


def test_struct_layouts_match_c():
    sizes, offs = _c_layout()
    assert sizes == [ctypes.sizeof(nat.ProblemDesc), ctypes.sizeof(nat.ProblemInfo), ctypes.sizeof(nat.SolverParamsC),
                     ctypes.sizeof(nat.Scalars), ctypes.sizeof(nat.CheckResult), ctypes.sizeof(nat.ShardDesc),
                     ctypes.sizeof(nat.SetupInfo)]
    assert offs == [nat.ProblemDesc.con_hi.offset, nat.CheckResult.xr_qd_inf.offset, nat.Scalars.have_avg_prev.offset,
                    nat.ProblemDesc.shard.offset, nat.ShardDesc.yw.offset, nat.SetupInfo.diag_bound.offset]


def test_product_fails_loudly_without_device(monkeypatch):
    """No silent host fallback: without CUDA the solve entry point raises."""
    import torch

    import paper_2602_23967_b200 as aq
    from paper_2602_23967_b200.errors import DeviceError

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    from paper_2602_23967_b200 import device

    monkeypatch.setattr(device, "_contexts", {})
    p = aq.random_qp(5, 3, "sparse", seed=1)
    with pytest.raises(DeviceError):
        aq.solve(p)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_23967_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.sub(r'(""".*?"""|#.*)', "", src, flags=re.S), fn

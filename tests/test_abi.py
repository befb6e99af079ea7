"""CPU-side checks of the C-ABI library (no GPU needed): it builds and loads, exports every
symbol include/rk_b200.h declares, and its host-only logic (partition rule, Butcher tableau,
step-size controller) agrees with the independently written oracle / input generators."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle
import rk_inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rk():
    from paper_2309_05331_b200 import build
    build.build()
    import paper_2309_05331_b200 as rk
    return rk


def header_functions():
    src = open(os.path.join(ROOT, "include", "rk_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rk_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(rk):
    L = ctypes.CDLL(rk.lib()._name)
    names = header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    from paper_2309_05331_b200._native import SIGNATURES
    assert sorted(SIGNATURES) == names     # the binding declares exactly the header's API


def test_abi_version(rk):
    assert rk.lib().rk_abi_version() == 5


@pytest.mark.parametrize("n,world", [(8, 2), (7, 2), (512, 24), (512, 8), (13, 13), (1, 1)])
def test_partition_matches_input_generator(rk, n, world):
    assert [rk.partition(n, world, r) for r in range(world)] == rk_inputs.slab_partition(n, world)


def test_partition_rejects_empty_ranks(rk):
    with pytest.raises(rk.RKError) as e:
        rk.partition(3, 4, 3)
    assert e.value.status == "RK_ERR_ARG"


@pytest.mark.parametrize("name", ["euler", "rk4", "cash_karp54", "dopri5", "rkf78", "midpoint",
                                  "modified_midpoint"])
def test_tableau_bitwise_equal_to_oracle(rk, name):
    lt = rk.tableau(name)
    ot = oracle.tableau(oracle.SCHEMES[name])
    s = ot["s"]
    assert lt["s"] == s and lt["order"] == ot["order"] and lt["err_order"] == ot["err_order"]
    for i in range(s):
        for j in range(s):
            f = ot["a"][i][j]
            assert lt["a"][i][j] == (f.numerator / f.denominator if f else 0.0)
        assert lt["b"][i] == ot["b"][i].numerator / ot["b"][i].denominator
        e = ot["b"][i] - ot["bhat"][i] if ot["err_order"] else 0
        want = (e.numerator / e.denominator) if e else 0.0
        assert lt["e"][i] == want, (name, i)
        assert lt["c"][i] == ot["c"][i].numerator / ot["c"][i].denominator


def test_controller_bitwise_equal_to_oracle(rk):
    rng = np.random.default_rng(11)
    Es = list(10.0 ** rng.uniform(-12, 4, 2000)) + [0.0, 0.5, 1.0, 1.0 + 2 ** -52, 5.0 ** -5, 1e300]
    for scheme, p, q in (("cash_karp54", 5, 4), ("dopri5", 5, 4), ("rkf78", 8, 7)):
        for E in Es:
            dt = float(rng.uniform(1e-3, 10.0))
            assert rk.controller(scheme, E, dt) == oracle.controller(E, dt, p, q), (E, dt)


def test_spec_controller_bitwise_equal_to_oracle(rk):
    """RK_OPT_CONTROLLER = 1 (R-28): the library's SPEC step adjuster equals the
    oracle's (pinned in test_oracle_spec_controller.py) bit for bit."""
    rng = np.random.default_rng(12)
    Es = list(10.0 ** rng.uniform(-12, 4, 2000)) + [0.0, 0.5, 1.0, 1.0 + 2 ** -52, 1e-300, 1e300]
    for scheme, p in (("cash_karp54", 5), ("dopri5", 5), ("rkf78", 8)):
        for E in Es:
            dt = float(rng.uniform(1e-3, 10.0))
            assert rk.controller(scheme, E, dt, kind=1) == oracle.controller_spec(E, dt, p), (E, dt)


def test_controller_errors(rk):
    with pytest.raises(rk.RKError) as e:
        rk.controller("rk4", 0.5, 1.0)
    assert e.value.status == "RK_ERR_UNSUPPORTED"
    with pytest.raises(rk.RKError) as e:
        rk.controller("dopri5", math.nan, 1.0)
    assert e.value.status == "RK_ERR_DIVERGED"


def test_no_gpu_is_a_loud_error(rk):
    """Without a usable GPU the library refuses (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rk.RKError) as e:
        rk.Context()
    assert e.value.status == "RK_ERR_CUDA"


def test_only_test_infrastructure_touches_oracle():
    """oracle/ is test infrastructure: outside tests/, only __graft_entry__.py (smoke) and
    bench.py (cpu_baseline / --impl reference) may import it."""
    allowed = {"__graft_entry__.py", "bench.py"}
    for dirpath, dirs, files in os.walk(ROOT):
        rel = os.path.relpath(dirpath, ROOT)
        if rel.split(os.sep)[0] in ("tests", "oracle", ".git", "build", "gpurun_out", "baseline"):
            dirs[:] = []
            continue
        for f in files:
            if f.endswith(".py") and f not in allowed:
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, os.path.join(rel, f)


def test_product_never_imports_oracle():
    """The product package shares no code with oracle/ (DESIGN.md §Boundary)."""
    pkg = os.path.join(ROOT, "paper_2309_05331_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "rk_oracle", "liboracle"):
                    assert bad not in txt, (f, bad)


def test_context_argument_validation(rk):
    """world > 1 needs either the NCCL unique id or a process group for the P2P handle
    exchange; an id of the wrong size is refused -- all before any device call."""
    with pytest.raises(ValueError):
        rk.Context(0, 2, 0)
    with pytest.raises(ValueError):
        rk.Context(0, 2, 0, unique_id=b"short")


def test_option_ids_match_header(rk):
    """The binding's option constants equal the header's rk_option values."""
    import re
    hdr = open(os.path.join(ROOT, "include", "rk_b200.h")).read()
    vals = {m.group(1): int(m.group(2)) for m in re.finditer(r"^\s*RK_OPT_(\w+)\s*=\s*(\d+)", hdr, re.M)}
    for name, v in vals.items():
        assert getattr(rk, "OPT_" + name) == v, name

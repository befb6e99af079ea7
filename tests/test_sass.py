"""Static checks of the built library's SASS (cuobjdump, no GPU needed): the stage kernels of
the headline (DOPRI5 adaptive) and RK4 paths load through TMA (UTMALDG) and keep their state in
registers -- no local-memory traffic (STL/LDL), which once crept in through code growth and
cost the FSAL tail stage 40 %."""
import os
import re
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2309_05331_b200", "librkb200.so")

pytestmark = pytest.mark.skipif(not (shutil.which("cuobjdump") and os.path.exists(LIB)),
                                reason="needs cuobjdump and the built library")


def _sass():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, name, body = {}, None, []
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if name:
                funcs[name] = "\n".join(body)
            name, body = m.group(1), []
        elif name:
            body.append(line)
    if name:
        funcs[name] = "\n".join(body)
    return funcs


@pytest.fixture(scope="module")
def sass():
    return _sass()


def _stage(sass, s, ad, i):
    key = f"gs_stage_kernelILi{s}ELi{ad}ELi{i}E"
    hits = [v for k, v in sass.items() if key in k]
    assert len(hits) == 1, key
    return hits[0]


# DOPRI5 adaptive try: k1 (first try only), stages 1..4, EPART stage 5, FSAL tail; RK4 stages
# (DOPRI5 adaptive stage 4 is the write-ahead stage, 5 the final combination it feeds)
HOT = [(1, 0, 0), (3, 0, 1), (3, 0, 2), (3, 0, 3), (3, 1, 4), (3, 1, 5), (3, 1, 6),
       (1, 0, 1), (1, 0, 2), (1, 0, 3), (0, 0, 0), (5, 0, 1), (3, 0, 4), (3, 0, 5),
       # the write-ahead stages before the K8 fixed-step tail pair (Y_{L-1}, Z_L, W)
       (2, 5, 3), (3, 5, 3), (4, 5, 10)]


@pytest.mark.parametrize("s,ad,i", HOT)
def test_hot_stage_kernels_use_tma_and_no_local_memory(sass, s, ad, i):
    body = _stage(sass, s, ad, i)
    assert "UTMALDG.4D" in body
    assert not re.search(r"\b(STL|LDL)\b", body), "local-memory traffic in a hot stage kernel"


def test_no_fma_contraction_in_stencil_arithmetic(sass):
    """R-17: the Gray–Scott stage arithmetic is DADD/DMUL only; DFMA appears only inside the
    IEEE division sequence of the error-ratio stages, never in k-only stages."""
    for (s, ad, i) in [(1, 0, 0), (1, 0, 1), (3, 0, 2), (0, 0, 0)]:
        assert "DFMA" not in _stage(sass, s, ad, i), (s, ad, i)


@pytest.mark.parametrize("s", [0, 1, 2, 3, 5])
def test_persistent_small_grid_kernel(sass, s):
    """K5 (rk_smallgrid.cu), configs[2]'s path: registers only and no FMA contraction (R-17)
    in the Euler / RK4 / Cash–Karp / DOPRI5 / midpoint instances (RKF78's spills 32 B)."""
    hits = [v for k, v in sass.items() if f"gs_coop_kernelILi{s}E" in k]
    assert len(hits) == 1
    assert not re.search(r"\b(STL|LDL)\b", hits[0])
    assert "DFMA" not in hits[0]


# K8 stage pairs (rk_pair.cu): <U1, WIN, BA, YOUT, DP> instances of the RK4 pairs, the explicit
# midpoint and the DOPRI5 tail pair -- TMA-fed, registers only (they sit at the 128-register cap
# of two 256-thread CTAs per SM, where a spill is the first thing to regress), no FMA in the k-only
# pairs (the DOPRI5 tail's IEEE division may use DFMA)
K8 = [("0", "0", "1", "1", "0", "0", "0", "0"), ("1", "1", "1", "0", "0", "0", "0", "0"),
      ("0", "0", "0", "0", "0", "0", "0", "0"), ("1", "1", "1", "0", "1", "0", "0", "0"),
      ("0", "0", "0", "0", "0", "0", "1", "1"),
      ("1", "1", "0", "0", "0", "0", "0", "0")]  # PAIR_LAST_NOA (Cash–Karp's fixed-step tail, b_5 = 0)


@pytest.mark.parametrize("flags", K8, ids=lambda f: "".join(f))
def test_k8_pair_kernels(sass, flags):
    key = "gs_pair_kernelI" + "".join(f"Lb{b}E" for b in flags) + "E"
    hits = [v for k, v in sass.items() if key in k]
    assert len(hits) == 1, key
    body = hits[0]
    assert "UTMALDG.4D" in body
    assert not re.search(r"\b(STL|LDL)\b", body), "local-memory traffic in a K8 pair kernel"
    if flags[4] == "0":
        assert "DFMA" not in body
# (the DOPRI5 tail pair's device-loop instance, dt read on the device, is not guarded: it runs
# inside the CUDA-graph try loop only)

"""CPU-side checks of the C ABI library: it loads and exports every symbol
include/greenllm.h declares, and ctypes layouts match the header."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "greenllm.h")


@pytest.fixture(scope="module")
def built():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2412_20322_b200 import native
    return native


def declared_functions():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:gl_status|int32_t|const char \*)\s*(gl_\w+)\s*\(",
                                 src, re.M)))


def test_header_declares_expected_calls():
    assert declared_functions() == sorted(["gl_eval_grid", "gl_eval_grid_sched",
                                           "gl_argmin_feasible", "gl_evaluate_host",
                                           "gl_evaluate_host_sched", "gl_link_demand",
                                           "gl_savings_surface",
                                           "gl_complete_matrices", "gl_argmin_matrices",
                                           "gl_last_launch_count",
                                           "gl_profile_enable", "gl_kernel_times",
                                           "gl_kernel_timeline",
                                           "gl_strerror", "gl_version"])


def test_library_exports_every_declared_symbol(built):
    lib = built.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", built.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), name
    assert set(built.EXPORTS) == set(declared_functions())


def test_version_and_strerror_without_gpu(built):
    lib = built.lib()
    assert lib.gl_version() == 3
    assert lib.gl_strerror(0) == b"ok"
    assert b"invalid" in lib.gl_strerror(-1)


def test_struct_layouts_match_header(built):
    """Compile a tiny C program against the header and compare sizeof/offsetof."""
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "greenllm.h"
int main(void){
 printf("%zu %zu %zu %zu %zu\n", sizeof(gl_trace), sizeof(gl_chain), sizeof(gl_chain_stats),
        sizeof(gl_scenario), sizeof(gl_grid));
 printf("%zu %zu %zu %zu\n", offsetof(gl_chain, alpha), offsetof(gl_chain, t1_us),
        offsetof(gl_chain, ttft_slo_us), offsetof(gl_chain, ce_old_g));
 printf("%zu %zu\n", offsetof(gl_chain_stats, req_hash), offsetof(gl_chain_stats, status));
 printf("%zu %zu %zu\n", sizeof(gl_link_params), sizeof(gl_link_stats),
        offsetof(gl_link_stats, peak_t_us));
 printf("%zu %zu %zu\n", sizeof(gl_savings_pair), sizeof(gl_savings),
        offsetof(gl_savings, eq4_energy_less));
 printf("%zu %zu\n", sizeof(gl_schedule), offsetof(gl_schedule, first_hi));
 return 0;}
"""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        open(src, "w").write(prog)
        exe = os.path.join(d, "l")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, src])
        lines = subprocess.check_output([exe], text=True).split("\n")
    sizes = list(map(int, lines[0].split()))
    N = built
    assert sizes == [C.sizeof(N.GlTrace), C.sizeof(N.GlChain), N.STATS_DTYPE.itemsize,
                     C.sizeof(N.GlScenario), C.sizeof(N.GlGrid)]
    offs = list(map(int, lines[1].split()))
    assert offs == [N.GlChain.alpha.offset, N.GlChain.t1_us.offset, N.GlChain.ttft_slo_us.offset,
                    N.GlChain.ce_old_g.offset]
    so = list(map(int, lines[2].split()))
    assert so == [N.STATS_DTYPE.fields["req_hash"][1], N.STATS_DTYPE.fields["status"][1]]
    lo = list(map(int, lines[3].split()))
    assert lo == [C.sizeof(N.GlLinkParams), N.LINK_DTYPE.itemsize,
                  N.LINK_DTYPE.fields["peak_t_us"][1]]
    sv = list(map(int, lines[4].split()))
    assert sv == [C.sizeof(N.GlSavingsPair), N.SAVINGS_DTYPE.itemsize,
                  N.SAVINGS_DTYPE.fields["eq4_energy_less"][1]]
    sc = list(map(int, lines[5].split()))
    assert sc == [C.sizeof(N.GlSchedule), N.GlSchedule.first_hi.offset]


def test_calls_fail_loudly_without_gpu(built):
    """No CPU fallback: on a GPU-less box a compute call returns an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2412_20322_b200.inputs import build_config
    g = build_config(1)
    tr = built.GlTrace(16, 16, 16, 1)
    ch = built.GlChain()
    ch.batch_cap, ch.max_prompt = 1, 1
    for f in ("t1_us", "e1_new_uj", "t2_us", "b2_old_us", "e2_old_uj", "step_us",
              "step_busy_new_us", "step_busy_old_us", "step_e_new_uj", "step_e_old_uj"):
        setattr(ch, f, 16)
    with pytest.raises(built.GreenLLMError):
        built.eval_grid([tr], [ch], 16, None, 0)
    with pytest.raises(built.GreenLLMError):  # the launch-order hint changes nothing here
        built.eval_grid([tr], [ch], 16, None, 0, sched=(0, 1))
    with pytest.raises(built.GreenLLMError) as ei:  # a bad hint is caught before the device
        built.eval_grid([tr], [ch], 16, None, 0, sched=(0, 2))
    assert ei.value.status == built.GL_E_INVALID
    with pytest.raises(built.GreenLLMError):
        built.link_demand([tr], [ch], [(4, 100)], 1_000_000, None, 16, 0)
    # host validation precedes the device check: a bad window is GL_E_INVALID, a
    # negative payload GL_E_DOMAIN
    with pytest.raises(built.GreenLLMError) as ei:
        built.link_demand([tr], [ch], [(4, 100)], 0, None, 16, 0)
    assert ei.value.status == built.GL_E_INVALID
    with pytest.raises(built.GreenLLMError) as ei:
        built.link_demand([tr], [ch], [(-1, 100)], 10, None, 16, 0)
    assert ei.value.status == built.GL_E_DOMAIN
    ch.ce_new_g, ch.ce_old_g = 1.0, 0.0
    scen = [[261.0, 1.0, 1.0]]
    with pytest.raises(built.GreenLLMError):  # no device
        built.savings_surface(16, [ch], [(0, 0)], scen, 16, 0)
    with pytest.raises(built.GreenLLMError) as ei:
        built.savings_surface(16, [ch], [(0, 1)], scen, 16, 0)
    assert ei.value.status == built.GL_E_LOOKUP
    with pytest.raises(built.GreenLLMError) as ei:
        built.savings_surface(16, [ch], [(0, 0)], [[261.0, 0.0, 1.0]], 16, 0)
    assert ei.value.status == built.GL_E_DOMAIN
    cm = built.complete_matrices
    with pytest.raises(built.GreenLLMError):  # no device
        cm(16, 16, 1, 4, 3, 2, 0.1, 10, 16, 0.0, 1.0, 16, None, None, 16, 0)
    for bad, code in (((16, 16, 1, 4, 3, 4, 0.1, 10), built.GL_E_INVALID),   # rank > cols
                      ((16, 16, 1, 4, 3, 9, 0.1, 10), built.GL_E_INVALID),   # rank > GL_MAX_RANK
                      ((16, 16, 1, 4, 2000, 2, 0.1, 10), built.GL_E_INVALID),
                      ((16, 16, 1, 4, 3, 2, -1.0, 10), built.GL_E_DOMAIN)):
        with pytest.raises(built.GreenLLMError) as ei:
            cm(*bad, 16, 0.0, 1.0, 16, None, None, 16, 0)
        assert ei.value.status == code


def test_oracle_and_product_share_no_code():
    """The oracle never includes the product header or sources, and vice versa."""
    osrc = open(os.path.join(ROOT, "oracle", "greenllm_oracle.c")).read()
    includes = re.findall(r'#include\s*[<"]([^>"]+)[>"]', osrc)
    assert set(includes) <= {"math.h", "stdint.h", "stdlib.h", "string.h"}, includes
    opy = open(os.path.join(ROOT, "oracle", "oracle.py")).read()
    assert "import paper_2412_20322_b200" not in opy and "from paper_2412_20322_b200" not in opy
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2412_20322_b200")):
        for f in files:
            if f.endswith(".py"):
                s = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in s and "import oracle" not in s, f
    cu = open(os.path.join(ROOT, "paper_2412_20322_b200", "csrc", "greenllm.cu")).read()
    assert "oracle" not in cu

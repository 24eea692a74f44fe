"""C-ABI checks that need no GPU: the library loads, exports every entry point that
include/rapid.h declares, and the ctypes structs match the C layout byte for byte."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rapid.h")
LIB = os.path.join(ROOT, "paper_1704_02083_b200", "librapid.so")


def _declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*\*?(rapid_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", ROOT, "lib"], check=True)
    return LIB


def test_library_exports_every_declared_symbol(built):
    names = _declared()
    assert len(names) >= 10
    nm = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (rapid_\w+)", nm))
    assert set(names) <= exported, set(names) - exported
    lib = ctypes.CDLL(built)  # loads without a GPU
    for n in names:
        assert hasattr(lib, n)


def test_binding_struct_layout_matches_header(built, tmp_path):
    import paper_1704_02083_b200 as rb
    prog = tmp_path / "layout.c"
    prog.write_text(r'''
#include <stdio.h>
#include <stddef.h>
#include "rapid.h"
int main(void) {
  printf("%zu %zu %zu %zu\n", sizeof(rapid_params), sizeof(rapid_sp_stat), sizeof(rapid_run_info), sizeof(rapid_profile));
  printf("%zu %zu %zu %zu %zu %zu %zu\n", offsetof(rapid_params, lambda_pos_q16), offsetof(rapid_params, proto_rgb),
         offsetof(rapid_params, tau2), offsetof(rapid_params, stats_mode), offsetof(rapid_run_info, phase),
         offsetof(rapid_params, feat_w_q16), sizeof(rapid_quality_result));
  return 0;
}
''')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    sizes = list(map(int, out[:4]))
    offs = list(map(int, out[4:]))
    assert sizes == [ctypes.sizeof(rb.rapid_params), ctypes.sizeof(rb.rapid_sp_stat),
                     ctypes.sizeof(rb.rapid_run_info), ctypes.sizeof(rb.rapid_profile)]
    assert offs == [rb.rapid_params.lambda_pos_q16.offset, rb.rapid_params.proto_rgb.offset,
                    rb.rapid_params.tau2.offset, rb.rapid_params.stats_mode.offset,
                    rb.rapid_run_info.phase.offset, rb.rapid_params.feat_w_q16.offset,
                    ctypes.sizeof(rb.rapid_quality_result)]


def test_init_without_gpu_fails_loudly(built):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1704_02083_b200 as rb
    with pytest.raises(rb.RapidError):
        rb.Rapid(0, 1024, 16)


def test_param_validation_happens_before_launch(built):
    """rapid_segment on a NULL ctx / bad params returns RAPID_E_ARG without touching a GPU."""
    import paper_1704_02083_b200 as rb
    lib = rb.lib
    p = rb.rapid_params()
    assert lib.rapid_segment(None, None, 8, 8, ctypes.byref(p), None, None) == -1
    assert lib.rapid_stats(None, None, 0, None) == -1
    assert rb.rapid_status_string(-6) == "RECOUNT integrity check failed"


def test_params_struct_has_no_implicit_padding():
    """Every byte of rapid_params belongs to a named field (the padding is explicit), so a
    C caller that fills it field by field cannot leave junk bytes that the graph-cache key
    would see."""
    import paper_1704_02083_b200 as rb
    total = sum(ctypes.sizeof(t) for _, t in rb.rapid_params._fields_)
    assert total == ctypes.sizeof(rb.rapid_params)

"""The C-ABI library loads, exports every symbol include/hetbridge.h declares,
and follows the status convention (ErrorCode ordinal + 1). No compute calls."""
import ctypes
import os
import re

from helpers import ROOT
from paper_2605_27678_b200 import _lib


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hetbridge.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == syms


def test_status_convention_matches_reference_error_codes():
    L = _lib.lib()
    names = ["RankOutOfModule", "CoordOutOfBounds", "IndivisibleBatch", "PartialOverlap", "NonIntegerFan",
             "PlanInfeasible", "ShardIntervalMismatch", "MissingSourceShard", "GradIntervalMismatch",
             "UnknownMicrobatch"]
    for i, n in enumerate(names):
        assert L.hb_error_name(i + 1).decode() == n
    assert L.hb_error_name(0).decode() == "OK"
    assert L.hb_error_name(25).decode() == "CudaError"
    assert L.hb_abi_version() == 7


def test_error_message_and_no_exception_across_abi():
    L = _lib.lib()
    lay = _lib.Layout(b"enc", 4, 1, 1, 2, 8)
    c = (ctypes.c_int * 4)()
    st = L.hb_coord_of_rank(ctypes.byref(lay), 7, c)
    assert st == 1
    assert "outside module 'enc'" in _lib.last_error()
    assert L.hb_coord_of_rank(None, 0, c) == 24  # null layout -> InvalidArgument


def test_exec_create_validates_before_touching_cuda():
    L = _lib.lib()
    e = _lib.Edge(_lib.Layout(b"a", 1, 1, 1, 2, 0), _lib.Layout(b"b", 1, 1, 1, 2, 0), 2, 4)
    p = ctypes.c_void_p()
    assert L.hb_plan_create(ctypes.byref(e), ctypes.byref(p)) == 0
    x = ctypes.c_void_p()
    m = (ctypes.c_int * 2)(0, 0)
    st = L.hb_exec_create(p, None, 0, 0, m, 2, None, ctypes.byref(x))  # n_gpus = 0
    assert st == 24 and not x.value
    L.hb_plan_destroy(p)


def test_header_has_no_cxx_or_torch_types():
    with open(os.path.join(ROOT, "include", "hetbridge.h")) as f:
        text = f.read()
    assert 'extern "C"' in text
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    for bad in ("std::", "torch", "at::", "c10", "template", "class "):
        assert bad not in text


C_CALLER = r"""
#include <stdio.h>
#include <string.h>
#include "hetbridge.h"
/* A plain C11 caller: the C2 edge through the C-ABI, no C++ and no CUDA calls. */
int main(void) {
  hb_edge e = {{"vit", 1, 1, 1, 8, 0}, {"llm", 4, 1, 1, 2, 0}, 64, 576 * 4096};
  int kind = -1, factor = -1, coord[4];
  if (hb_classify_dp_relation(&e, &kind, &factor)) return 1;
  hb_plan* p = NULL;
  if (hb_plan_create(&e, &p)) return 2;
  size_t n = 0;
  if (hb_plan_export(p, 2, NULL, 0, &n)) return 3;
  char buf[1 << 16];
  if (n >= sizeof buf || hb_plan_export(p, 2, buf, sizeof buf, &n)) return 4;
  if (hb_coord_of_rank(&e.dest, 5, coord)) return 5;
  int st = hb_coord_of_rank(&e.dest, 9, coord); /* outside the module: RankOutOfModule = 1 */
  char msg[256];
  hb_last_error(msg, sizeof msg);
  printf("%d %d %zu %d %d %d %s\n", kind, factor, n, coord[0], coord[3], st, hb_error_name(st));
  fputs(buf, stdout);
  hb_plan_destroy(p);
  return 0;
}
"""


def test_plain_c_caller_compiles_links_and_runs(tmp_path):
    """The boundary is a C ABI: a C11 program (gcc -std=c11 -pedantic -Werror)
    includes include/hetbridge.h, links libhetbridge.so and plans the C2 edge;
    its answers equal the Python face's."""
    import shutil
    import subprocess

    if not shutil.which("gcc"):
        pytest.skip("no C compiler")
    src = tmp_path / "caller.c"
    src.write_text(C_CALLER)
    exe = tmp_path / "caller"
    libdir = os.path.join(ROOT, "paper_2605_27678_b200")
    subprocess.run(["gcc", "-std=c11", "-pedantic", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-L", libdir, "-lhetbridge", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    head, text = out.split("\n", 1)
    kind, factor, n, tp, dp, st, name = head.split()
    from paper_2605_27678_b200 import bridge as hbb
    from paper_2605_27678_b200 import configs

    plan = hbb.plan_bridge(configs.get("c2").edge())
    assert text == hbb.export_plan(plan, 2) and int(n) == len(text)
    assert (int(factor), int(tp), int(dp)) == (4, 1, 1)  # FanIn k=4; rank 5 = (tp 1, dp 1)
    assert int(st) == 1 and name == "RankOutOfModule"

"""The C ABI (include/gadi_b200.h) on the CPU: the in-tree library loads
without a GPU, exports every function the header declares, the ctypes
binding (_lib.py) declares the same set, and the binding's struct layouts
match the C compiler's.  Without a CUDA device the product path refuses to
run (there is no CPU fallback)."""

import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2512_21164_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "gadi_b200.h"


def _declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return set(re.findall(r"\b(gadi_\w+)\s*\(", text))


def test_header_functions_exported_and_bound(libpath):
    names = _declared()
    assert len(names) >= 30
    lib = C.CDLL(str(libpath))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)
    _lib.load()  # attaches every signature


def test_struct_layouts_match_c(tmp_path, libpath):
    src = tmp_path / "sizes.c"
    src.write_text(f'''#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(gadi_coef), sizeof(gadi_csr), sizeof(gadi_problem_desc),
         sizeof(gadi_outer_scalars), sizeof(gadi_inner_stats), sizeof(gadi_phase_times), sizeof(gadi_step_args),
         offsetof(gadi_problem_desc, u_s));
  return 0;
}}
''')
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(_lib.Coef), C.sizeof(_lib.Csr), C.sizeof(_lib.ProblemDesc), C.sizeof(_lib.OuterScalars),
            C.sizeof(_lib.InnerStats), C.sizeof(_lib.PhaseTimes), C.sizeof(_lib.StepArgs),
            _lib.ProblemDesc.u_s.offset]
    assert got == want


def test_build_info_and_error_string(libpath):
    lib = _lib.load()
    assert b"sm_100a" in lib.gadi_build_info()
    assert isinstance(lib.gadi_last_error(), bytes)


def test_no_cpu_fallback(libpath):
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    import paper_2512_21164_b200 as g

    with pytest.raises(_lib.GpuUnavailable):
        g.gadi_solve(g.build_cdr_2d(8), cfg=g.GadiConfig(alpha=1.0))
    with pytest.raises(_lib.GpuUnavailable):
        g.spmv(g.build_cdr_2d(8).A, [1.0] * 64, "fp64")

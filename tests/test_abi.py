"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol include/cc.h
declares, refuses to run without a GPU (no CPU fallback), and its one pure-host entry point
(cc_hmf) agrees with the oracle's HMF."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2604_18801_b200 as cc
from paper_2604_18801_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cc.h")).read()
    return sorted(set(re.findall(r"\b(cc_[a-z_0-9]+)\s*\(", src)))


def test_header_declarations_are_exported():
    lib = cc.lib()
    names = _declared()
    assert "cc_find_vulnerable" in names and "cc_correct" in names
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", cc.lib_path()], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), f"{n} not exported"
    assert set(binding.EXPORTS) == set(names)


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", cc.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = cc.lib()
    p = binding._Params()
    lib.cc_default_params(C.byref(p))
    h = C.c_void_p()
    st = lib.cc_create(C.byref(h), 0, None, C.byref(p), None)
    assert st == 68 and not h.value
    with pytest.raises(cc.CCError):
        cc.Corrector(cc.Params(xi=1e-3))


def test_default_params_are_the_papers():
    p = binding._Params()
    cc.lib().cc_default_params(C.byref(p))
    assert (p.eta, p.m, p.alpha, p.beta1, p.beta2, p.eps_adam, p.eps_loss) == (0.2, 16, 1e-3, 0.9, 0.999, 1e-8, 1e-10)


def test_cc_hmf_matches_oracle():
    rng = np.random.default_rng(1)
    sizes = np.sort((20 * rng.pareto(0.9, 500) + 20).astype(np.int64))[::-1]
    e1, d1 = cc.hmf(sizes, 8.0, 50)
    e2, d2 = oracle.hmf(sizes, 8.0, 50)
    assert np.allclose(e1, e2, rtol=0, atol=1e-12) and np.allclose(d1, d2, rtol=1e-12)
    e1, d1 = cc.hmf(sizes[:100], 8.0, 50, lo=e2[0], hi=e2[-1])
    e2, d2 = oracle.hmf(sizes[:100], 8.0, 50, lo=e2[0], hi=e2[-1])
    assert np.allclose(d1, d2, rtol=1e-12)


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of the ABI structs have the C compiler's sizes and field offsets."""
    structs = {"cc_params": binding._Params, "cc_dist": binding._Dist, "cc_vp_info": binding._VP,
               "cc_corr_info": binding._Corr, "cc_mcc_info": binding._Mcc, "cc_run_info": binding._Run,
               "cc_thresholds": binding._Th}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "cc.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", f"-I{os.path.join(ROOT, 'include')}", str(src), "-o", str(exe)])
    got = dict(ln.split() for ln in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, f"{cname}.{f}"

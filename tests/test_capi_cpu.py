"""CPU-side checks of the C-ABI boundary (no GPU needed): the library loads,
exports every function include/mgcuda.h declares, the ctypes struct mirrors
match the C layout, host-only helpers agree with the reference, and compute
entry points fail loudly (MG_ECUDA) instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2309_15676_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mgcuda.h")
LIB = os.path.join(ROOT, "paper_2309_15676_b200", "libmgcuda.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(mg_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2309_15676_b200", "csrc")],
                       check=True)
    from paper_2309_15676_b200 import _lib
    return _lib.load()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("mg_meta_update", "mg_adam_update", "mg_mt64_draw", "mg_minirender_sample_pair",
                 "mg_run_replicates", "mg_ctx_create"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_layouts_match_c():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "mgcuda.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(mg_experiment_config),
         sizeof(mg_moment2_scalars), sizeof(mg_meta_params), sizeof(mg_adam_scalars),
         sizeof(mg_update_scalars), sizeof(mg_meta_update_args), sizeof(mg_meta_extras),
         sizeof(mg_run_record), sizeof(mg_run_series), offsetof(mg_experiment_config, rng));
  return 0;
}
"""
    tmp = os.path.join(ROOT, "oracle", "_build")
    os.makedirs(tmp, exist_ok=True)
    c_path, exe = os.path.join(tmp, "abi_sizes.c"), os.path.join(tmp, "abi_sizes")
    with open(c_path, "w") as f:
        f.write(src)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c_path, "-o", exe], check=True)
    got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(_abi.ExperimentConfigC), C.sizeof(_abi.Moment2Scalars),
            C.sizeof(_abi.MetaParams), C.sizeof(_abi.AdamScalars), C.sizeof(_abi.UpdateScalars),
            C.sizeof(_abi.MetaUpdateArgs), C.sizeof(_abi.MetaExtras), C.sizeof(_abi.RunRecordC),
            C.sizeof(_abi.RunSeriesC), _abi.ExperimentConfigC.rng.offset]
    assert got == want


def test_host_helpers_match_reference(lib, oracle):
    for x in (0, 1, 2**63, 12345678901234567):
        assert lib.mg_mix64(x) == oracle.mix64(x)
    # Rng::stream seed (rng.hpp:23-25)
    seed = lib.mg_stream_seed(7, 3)
    assert seed == oracle.mix64(oracle.mix64(7) ^ (3 + 0x51ed2701e35f3a6d))


def test_config_defaults_and_validation(lib):
    c = _abi.ExperimentConfigC()
    lib.mg_config_defaults(C.byref(c))
    ref = _abi.config_from()
    for name, _ in _abi.ExperimentConfigC._fields_:
        assert getattr(c, name) == getattr(ref, name), name
    assert lib.mg_config_validate(C.byref(c)) == 0
    bad = [("lr", 0.0), ("beta_f", 1.0), ("beta_delta", -0.1), ("beta1", 1.0), ("beta2", 1.5),
           ("iterations", 0), ("replicates", 0), ("coord", -1), ("non_zero_centred", 1),
           ("problem", 7), ("optimizer", 3), ("trajectory", 5), ("diff_norm", 2)]
    for k, v in bad:
        c2 = _abi.ExperimentConfigC.from_buffer_copy(c)
        setattr(c2, k, v)
        assert lib.mg_config_validate(C.byref(c2)) == _abi.MG_EINVAL, k
    c3 = _abi.ExperimentConfigC.from_buffer_copy(c)
    c3.problem = 9
    lib.mg_config_validate(C.byref(c3))
    assert b"exp-rate" in lib.mg_last_error()  # valid set listed (test_harness.cpp:228-246)


def test_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = lib.mg_ctx_create(0, None, C.byref(h))
    assert rc == _abi.MG_ECUDA
    assert b"no CPU fallback" in lib.mg_last_error()


def test_python_config_mirror_rejects_unknown_names():
    with pytest.raises(ValueError, match="exp-rate"):
        _abi.config_from(problem="banana")
    with pytest.raises(ValueError, match="meta"):
        _abi.config_from(optimizer="sgd")

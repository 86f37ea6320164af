"""CPU checks of the C-ABI boundary: the library builds, loads and exports every
symbol include/nalar.h declares; struct layouts match; no compute on CPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nalar.h")


@pytest.fixture(scope="module")
def lib():
    # loaded by path: importing the package would load libnalar.so before it exists
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_nalar_build", os.path.join(ROOT, "paper_2601_05109_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.build_lib()


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|void\*|const char\*)\s+(nalar_\w+)\s*\(", txt,
                                 re.M)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 14
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib], text=True)
    exported = set(re.findall(r" T (nalar_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    from paper_2601_05109_b200 import nalar
    assert set(names) == set(nalar.EXPORTS)
    h = C.CDLL(lib)
    for n in names:
        getattr(h, n)


def test_sm100a_code_only(lib):
    out = subprocess.check_output(["cuobjdump", "-lelf", lib], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", lib], text=True)
    assert "UBLKCP" in sass            # K1 stages its table slice with TMA bulk copies
    for k in ("k0_validate", "k1_sweep", "k4_assign"):
        assert k in sass


def test_struct_layouts_match_header(lib):
    """Compile a tiny C probe against include/nalar.h and compare sizeof/offsetof
    with the ctypes mirrors in the binding."""
    from paper_2601_05109_b200 import nalar
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "nalar.h"
int main(void){
 printf("%zu %zu %zu %zu\n", sizeof(nalar_config), sizeof(nalar_snapshot), sizeof(nalar_decisions), sizeof(nalar_epoch_stats));
 printf("%zu %zu %zu\n", offsetof(nalar_config, flags), offsetof(nalar_snapshot, t_affinity), offsetof(nalar_decisions, n_assigned));
 return 0;}
'''
    tmp = os.path.join(ROOT, "build")
    os.makedirs(tmp, exist_ok=True)
    src, exe = os.path.join(tmp, "probe.c"), os.path.join(tmp, "probe")
    open(src, "w").write(probe)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe])
    l1, l2 = subprocess.check_output([exe], text=True).split("\n")[:2]
    sizes = [int(x) for x in l1.split()]
    offs = [int(x) for x in l2.split()]
    assert sizes == [C.sizeof(nalar.nalar_config), C.sizeof(nalar.nalar_snapshot),
                     C.sizeof(nalar.nalar_decisions), C.sizeof(nalar.nalar_epoch_stats)]
    assert offs == [nalar.nalar_config.flags.offset, nalar.nalar_snapshot.t_affinity.offset,
                    nalar.nalar_decisions.n_assigned.offset]


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    from paper_2601_05109_b200 import nalar
    assert nalar.nalar_abi_version() == 2
    cfg = nalar.nalar_config()
    cfg.world, cfg.max_futures, cfg.max_edges, cfg.max_workflows = 1, 10, 10, 2
    cfg.max_instances, cfg.max_types = 2, 1
    assert nalar.nalar_workspace_bytes(cfg) > 0
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    with pytest.raises(nalar.NalarError) as ei:
        nalar.nalar_create(cfg)
    assert ei.value.code == nalar.NALAR_E_CUDA


def test_bad_limits_rejected(lib):
    from paper_2601_05109_b200 import nalar
    cfg = nalar.nalar_config()
    cfg.world, cfg.max_types, cfg.levels = 1, 65, 256       # > NALAR_MAX_TYPES
    with pytest.raises(nalar.NalarError) as ei:
        nalar.nalar_create(cfg)
    assert ei.value.code == nalar.NALAR_E_INVAL

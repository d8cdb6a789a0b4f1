"""-m "not gpu": the C-ABI library loads, exports every symbol include/pariskv.h declares, and its host-side
logic (Prop. 1 constants, schedule, argument validation) agrees with the independent oracle. No compute."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import synth
from oracle import coarse, levels

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pkv():
    from paper_2602_07721_b200 import build
    build.build()
    from paper_2602_07721_b200 import pariskv
    return pariskv


def header_functions():
    src = open(os.path.join(ROOT, "include", "pariskv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:pkv_status|const char\*)\s+([a-z_][a-z0-9_]*)\s*\(", src)))


def test_every_declared_symbol_is_exported(pkv):
    names = header_functions()
    assert len(names) >= 18
    lib = ctypes.CDLL(pkv.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(pkv.EXPORTED)


def test_sm100a_cubin_in_library(pkv):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkv.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_prop1_constants_bit_identical_to_oracle(pkv):
    cfg = pkv.config_init(32, 8, synth.rotation_sign_bits())
    L = np.array(cfg.mag_levels[:], dtype=np.float32)
    assert np.array_equal(L, levels.levels_f32(8))
    assert np.array_equal(np.array(cfg.mag_mid_sq[:]), levels.mid_sq(levels.levels_f32(8)))
    assert list(cfg.tier_bonus[:6]) == [6, 5, 4, 3, 2, 1] and cfg.n_tiers == 6
    assert list(cfg.rot_sign[:]) == list(synth.rotation_sign_bits())


@pytest.mark.parametrize("n", [1, 50, 99, 100, 4096, 19999, 20000, 32496, 59999, 60000, 130800, 199999, 200000,
                               1048304, 5_000_000])
@pytest.mark.parametrize("k", [1, 64, 100])
def test_schedule_matches_oracle(pkv, n, k):
    assert pkv.schedule(n, k) == coarse.schedule(n, k)


def test_config_validation(pkv):
    with pytest.raises(pkv.PkvError):
        pkv.config_init(32, 5, synth.rotation_sign_bits())      # n_q % n_kv != 0
    with pytest.raises(pkv.PkvError):
        pkv.config_init(64, 8, synth.rotation_sign_bits())      # GQA group 8 > 4
    with pytest.raises(pkv.PkvError):
        pkv.schedule(-1, 10)


def test_index_create_fails_cleanly_without_gpu(pkv):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = pkv.config_init(32, 8, synth.rotation_sign_bits())
    with pytest.raises(pkv.PkvError) as e:
        pkv.Index(cfg, 1, 1024)
    assert e.value.status in (pkv.PKV_ERR_CUDA, pkv.PKV_ERR_INVALID_ARG)


def test_no_predecessor_output_read_before_griddepcontrol_wait(pkv):
    """Programmatic dependent launch contract, checked on the SASS of the built kernels: before
    griddepcontrol.wait (ACQBULK) a kernel may only load data no kernel of the decode chain writes — the
    index's centroid ids (scan prefetch), the caller's hot rows (qprep, attend_partial, fused top-k) and the
    query (fused top-k) — and may not store. A predecessor output read there (e.g. a const __restrict__ load the compiler
    hoisted onto the non-coherent path) is a race that returns stale candidates."""
    import importlib.util
    import shutil
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    spec = importlib.util.spec_from_file_location("check_pdl_sass", os.path.join(ROOT, "scripts", "check_pdl_sass.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    build_dir = os.path.join(ROOT, "paper_2602_07721_b200", "build")
    res = {}
    for f in ("qprep.cu.o", "scan.cu.o", "rerank.cu.o", "attend.cu.o", "postings.cu.o"):
        res.update(mod.prewait_loads(os.path.join(build_dir, f)))
    assert len(res) >= 10, sorted(res)

    def ops(v):
        return [x.split()[1] if x.startswith("@") else x.split()[0] for x in v]

    for name, v in res.items():
        kinds = ops(v)
        assert all(k.startswith("LDG") for k in kinds), (name, v)  # no stores / atomics before the wait
        if "scan_kernel" in name:
            assert set(kinds) <= {"LDG.E.NA.128.CONSTANT"} and len(kinds) <= 4, (name, v)  # centroid-id rows
        elif "qprep_kernel" in name:
            assert set(kinds) <= {"LDG.E.64"} and len(kinds) <= 16, (name, v)  # hot K/V rows only
        elif "attend_partial_kernel" in name:
            assert set(kinds) <= {"LDG.E.64"}, (name, v)  # query + hot rows
        elif "topk_cl_kernelILb1" in name:
            assert set(kinds) <= {"LDG.E.64"}, (name, v)  # the query and the caller's hot rows
        else:
            assert kinds == [], (name, v)

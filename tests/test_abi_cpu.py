"""CPU-side checks of the C-ABI library (no GPU): it builds for sm_100a, loads,
exports every symbol include/libboris.h declares, and its host-only logic
(argument validation, status strings, field-handle validation, no-device
errors) behaves as documented.  Also: AoS record layout = the paper's struct,
and the oracle / CUDA path independence rules."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "libboris.h")


@pytest.fixture(scope="module")
def lb():
    from paper_2104_04579_b200 import _build
    _build.build()
    import paper_2104_04579_b200 as lb
    lb.load_library()
    return lb


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(boris_[a-z0-9_]+)\s*\(", src))


def test_library_exports_every_declared_symbol(lb):
    declared = header_functions()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", lb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (boris_[a-z0-9_]+)", out))
    assert declared <= exported, declared - exported
    assert declared == set(lb.EXPORTED)
    lib = lb.load_library()
    for name in declared:
        getattr(lib, name)


def test_library_is_sm100a(lb):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lb.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_sass_evidence(lb):
    """The compiled sm_100a code uses what DESIGN.md claims: 128-bit streaming loads
    (LDG.E.128), evict-first stores (STG.E.EF.128), TMA bulk copies with mbarrier
    transaction counting (UBLKCP, SYNCS.ARRIVE.TRANS64) and MUFU rsqrt."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lb.LIB_PATH],
                          capture_output=True, text=True, check=True).stdout
    for op in ("LDG.E.NA.128", "LDG.E.NA.128.CONSTANT", "STG.E.EF.128", "UBLKCP.S.G",
               "UBLKCP.G.S", "SYNCS.ARRIVE.TRANS64", "MUFU.RSQ", "MUFU.COS"):
        assert op in sass, op


def build_c_example(lb, tmp_path):
    exe = tmp_path / "push_c_abi"
    pkg = os.path.dirname(lb.LIB_PATH)
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "push_c_abi.c"), "-L", pkg, "-lboris",
                           f"-Wl,-rpath,{pkg}", "-lm", "-o", str(exe)])
    return exe


def test_c_example_links_against_the_abi(lb, tmp_path):
    """A plain C program compiles against include/libboris.h and links libboris.so;
    without a GPU it stops at boris_ensemble_create with BORIS_E_NO_DEVICE (exit 2)."""
    import torch
    exe = build_c_example(lb, tmp_path)
    if torch.cuda.is_available():
        pytest.skip("a GPU is present (tests/test_gpu_parity.py runs it)")
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 2, r.stdout + r.stderr
    assert "no CUDA device" in r.stdout


def test_abi_version_and_status_strings(lb):
    assert lb.boris_abi_version() == 1
    for code, name in [(0, "BORIS_OK"), (1, "BORIS_E_INVALID_ARG"), (5, "BORIS_E_MISMATCH"),
                       (7, "BORIS_E_NO_DEVICE"), (99, "BORIS_E_UNKNOWN")]:
        assert lb.boris_status_string(code) == name


def test_no_device_is_reported_not_faked(lb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_ensemble_create(0, lb.BORIS_LAYOUT_SOA, lb.BORIS_FP32, 10,
                                 [(-4.8e-10, 9.1e-28)], 3e10)
    assert ei.value.status == lb.BORIS_E_NO_DEVICE


def test_argument_validation_host_only(lb):
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_ensemble_create(0, 7, lb.BORIS_FP32, 10, [(1.0, 1.0)], 1.0)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_ensemble_create(0, lb.BORIS_LAYOUT_SOA, lb.BORIS_FP32, -1, [(1.0, 1.0)], 1.0)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:   # beyond BORIS_MAX_PARTICLES
        lb.boris_ensemble_create(0, lb.BORIS_LAYOUT_SOA, lb.BORIS_FP64,
                                 lb.BORIS_MAX_PARTICLES + 1, [(1.0, 1.0)], 1.0)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:   # mass must be > 0
        lb.boris_ensemble_create(0, lb.BORIS_LAYOUT_SOA, lb.BORIS_FP32, 1, [(1.0, 0.0)], 1.0)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:   # too many types
        lb.boris_ensemble_create(0, lb.BORIS_LAYOUT_SOA, lb.BORIS_FP32, 1, [(1.0, 1.0)] * 257, 1.0)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError) as ei:
        lb.boris_push(None, None, 1.0, 1)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    assert "NULL" in lb.boris_last_error()


def test_options_are_abi_calls_not_environment(lb):
    """boris_set_option / boris_get_option (host only, no device needed): defaults,
    round trip, validation.  The library reads no environment variables."""
    assert lb.boris_get_option(lb.BORIS_OPT_FUSED_GENERIC) == 0
    chunk0 = lb.boris_get_option(lb.BORIS_OPT_HOST_CHUNK)
    assert chunk0 == 4 << 20
    assert lb.boris_get_option(lb.BORIS_OPT_MD_ORDER) == 1
    try:
        lb.boris_set_option(lb.BORIS_OPT_MD_ORDER, 0)
        assert lb.boris_get_option(lb.BORIS_OPT_MD_ORDER) == 0
        lb.boris_set_option(lb.BORIS_OPT_FUSED_GENERIC, 1)
        assert lb.boris_get_option(lb.BORIS_OPT_FUSED_GENERIC) == 1
        lb.boris_set_option(lb.BORIS_OPT_HOST_CHUNK, 4096)
        assert lb.boris_get_option(lb.BORIS_OPT_HOST_CHUNK) == 4096
        for opt, bad in ((lb.BORIS_OPT_FUSED_GENERIC, 2), (lb.BORIS_OPT_HOST_CHUNK, 1023),
                         (lb.BORIS_OPT_MD_ORDER, -1), (99, 0)):
            with pytest.raises(lb.BorisError) as ei:
                lb.boris_set_option(opt, bad)
            assert ei.value.status == lb.BORIS_E_INVALID_ARG
        with pytest.raises(lb.BorisError):
            lb.boris_get_option(99)
    finally:
        lb.boris_set_option(lb.BORIS_OPT_FUSED_GENERIC, 0)
        lb.boris_set_option(lb.BORIS_OPT_HOST_CHUNK, chunk0)
        lb.boris_set_option(lb.BORIS_OPT_MD_ORDER, 1)
    # (the static CUDA runtime linked into libboris.so reads CUDA_* variables itself;
    # libboris' own sources never call getenv)
    import glob
    csrc = os.path.join(os.path.dirname(lb.LIB_PATH), "csrc")
    for f in glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cuh")):
        assert "getenv(" not in open(f).read(), f


def test_field_handles_validate(lb):
    f = lb.boris_field_create_uniform([1, 2, 3], [0, 0, 1])
    lb.boris_field_destroy(f)
    f = lb.boris_field_create_plane_wave(1.0, [1, 0, 0], [0, 1, 0], 2.0, 2.0, 0.1)
    lb.boris_field_destroy(f)
    with pytest.raises(lb.BorisError) as ei:   # e_hat not orthogonal to k_hat
        lb.boris_field_create_plane_wave(1.0, [1, 0, 0], [1, 0, 0], 2.0, 2.0)
    assert ei.value.status == lb.BORIS_E_INVALID_ARG
    with pytest.raises(lb.BorisError):         # not a unit vector
        lb.boris_field_create_plane_wave(1.0, [2, 0, 0], [0, 1, 0], 2.0, 2.0)
    with pytest.raises(lb.BorisError):
        lb.boris_field_create_uniform([float("inf"), 0, 0], [0, 0, 0])
    f = lb.boris_field_create_mdipole(1.0, 2.0, 3.0)
    lb.boris_field_destroy(f)
    with pytest.raises(lb.BorisError):
        lb.boris_field_create_mdipole(1.0, 2.0, 0.0)
    lb.boris_field_destroy(None)


def test_aos_record_layout_is_the_papers_struct(tmp_path):
    """Particle {FP3 position; FP3 momentum; FP weight; FP gamma;
    short type;} is 34 B -> 36 B aligned (float), 66 B -> 72 B (double)."""
    src = tmp_path / "rec.c"
    src.write_text(r'''
#include <stdio.h>
#include <stddef.h>
#include "libboris.h"
#define REC(FP, NAME) typedef struct { FP position[3]; FP momentum[3]; FP weight; FP gamma; short type; } NAME;
REC(float, P32)
REC(double, P64)
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(P32), offsetof(P32, momentum), offsetof(P32, weight),
         offsetof(P32, gamma), offsetof(P32, type), (size_t)BORIS_AOS_RECORD_BYTES_FP32);
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(P64), offsetof(P64, momentum), offsetof(P64, weight),
         offsetof(P64, gamma), offsetof(P64, type), (size_t)BORIS_AOS_RECORD_BYTES_FP64);
  return 0; }
''')
    exe = tmp_path / "rec"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    lines = subprocess.check_output([str(exe)], text=True).split("\n")
    assert lines[0].split() == ["36", "12", "24", "28", "32", "36"]
    assert lines[1].split() == ["72", "24", "48", "56", "64", "72"]


def test_oracle_and_cuda_path_share_nothing():
    """The oracle (test infra) and the product share no code; the product never
    imports the oracle."""
    pkg = os.path.join(ROOT, "paper_2104_04579_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, fn
                assert "boris_oracle" not in txt, fn
    for fn in os.listdir(os.path.join(ROOT, "oracle")):
        if fn.endswith((".c", ".h", ".py")):
            txt = open(os.path.join(ROOT, "oracle", fn)).read()
            assert not re.search(r"#include\s+[\"<](libboris|boris_device|boris_internal)", txt), fn
            assert not re.search(r"^\s*(import|from)\s+(paper_2104_04579_b200|synth)\b", txt,
                                 re.M), fn


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without libboris.so every call raises ImportError."""
    import subprocess
    import sys
    env = dict(os.environ, LIBBORIS_PATH=str(tmp_path / "absent" / "libboris.so"))
    r = subprocess.run([sys.executable, "-c",
                        "import paper_2104_04579_b200 as lb; lb.boris_abi_version()"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "no CPU fallback" in r.stderr

"""Host logic and the C-ABI boundary, on CPU (no compute calls)."""

import ctypes
import os
import re

import pytest

from paper_2504_19442_b200 import (AllocationError, ArgumentError, CollectiveFault,
                                   ConfigurationError, ProblemShape, ShmemError,
                                   SynchronizationFault, UsageError, WorldSpec, _lib)
from paper_2504_19442_b200 import errors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shmem_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(sh_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_lib.SIGNATURES)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.sh_version() >= 1
    assert lib.sh_ipc_handle_size() == 64


def test_load_rejects_a_second_library(tmp_path):
    lib = _lib.load()
    assert _lib.load(_lib.LIB_PATH if not os.environ.get("SHB_LIB") else
                     os.environ["SHB_LIB"]) is lib
    other = tmp_path / "libother.so"
    other.write_bytes(b"")
    with pytest.raises(ShmemError, match="already loaded"):
        _lib.load(str(other))


def test_argument_errors_without_gpu():
    lib = _lib.load()
    # argument validation precedes any CUDA work
    rc = lib.sh_set_tile_config(96, 2)
    assert rc == _lib.SH_ERR_ARG
    with pytest.raises(ArgumentError, match="bn must be"):
        _lib.check(rc)
    assert lib.sh_set_tile_config(0, 0) == _lib.SH_OK
    assert lib.sh_gemm(None, None, None, 0, 8, 8, 0, None, 0, None) == _lib.SH_ERR_ARG
    assert lib.sh_gemm(None, None, None, 8, 6, 8, 0, None, 0, None) == _lib.SH_ERR_ARG  # n % 8
    assert lib.sh_gemm(None, None, None, 8, 8, 8, 7, None, 0, None) == _lib.SH_ERR_ARG  # dtype
    lib.sh_gemm(None, None, None, 8, 6, 8, 0, None, 0, None)
    assert b"multiples of 8" in lib.sh_last_error()
    out = ctypes.c_void_p()
    assert lib.sh_world_create(0, None, 1 << 20, 0, 5.0, ctypes.byref(out)) == _lib.SH_ERR_CONFIG
    assert lib.sh_world_create(2, None, 0, 0, 5.0, ctypes.byref(out)) == _lib.SH_ERR_CONFIG


def test_status_codes_map_to_reference_taxonomy():
    for code, exc in [(_lib.SH_ERR_ARG, ArgumentError), (_lib.SH_ERR_ALLOC, AllocationError),
                      (_lib.SH_ERR_TIMEOUT, SynchronizationFault), (_lib.SH_ERR_STATE, UsageError),
                      (_lib.SH_ERR_CONFIG, ConfigurationError)]:
        with pytest.raises(exc):
            _lib.check(code)
    with pytest.raises(ShmemError):
        _lib.check(_lib.SH_ERR_CUDA)
    _lib.check(_lib.SH_OK)


def test_error_hierarchy_matches_reference():
    assert issubclass(errors.ArgumentError, ValueError)
    assert issubclass(errors.RangeError, errors.ArgumentError)
    cf = CollectiveFault("x", {2: ArgumentError("a"), 0: ArgumentError("b")})
    assert isinstance(cf.first, ArgumentError) and set(cf.failures) == {0, 2}


def test_problem_shape_validation():
    with pytest.raises(ArgumentError):
        ProblemShape(m=0, n=4, k=4)
    with pytest.raises(ArgumentError):
        ProblemShape(m=9, n=4, k=4).rows_per_rank(2)
    with pytest.raises(ArgumentError):
        ProblemShape(m=8, n=8, k=8, tile_m=-1)
    assert ProblemShape(m=8, n=8, k=8).rows_per_rank(4) == 2
    # the tensor-core path computes in bf16/fp16; int64 (the reference
    # default) and the other widened types are staged in bf16 when exact
    import numpy as np
    import torch

    s = ProblemShape(m=8, n=6, k=12)
    assert (s.io_dtype, s.widened, s.torch_dtype) == ("int64", True, torch.bfloat16)
    assert (s.k_padded, s.n_padded) == (16, 8)
    assert ProblemShape(m=8, n=8, k=8, dtype=np.float32).io_dtype == "float32"
    assert ProblemShape(m=8, n=8, k=8, dtype="bf16").torch_dtype == torch.bfloat16
    assert not ProblemShape(m=8, n=8, k=8, dtype="bf16").widened
    assert ProblemShape(m=8, n=8, k=8, dtype="float16").dtype_code == _lib.SH_DTYPE_FP16
    with pytest.raises(ArgumentError, match="bf16/fp16"):
        ProblemShape(m=8, n=8, k=8, dtype="complex64").torch_dtype


def test_serialising_tool_detection(monkeypatch):
    from paper_2504_19442_b200.core import serialising_tool

    for var in ("SHB_PHASED", "CUDA_INJECTION64_PATH", "CUDA_LAUNCH_BLOCKING"):
        monkeypatch.delenv(var, raising=False)
    assert not serialising_tool()
    monkeypatch.setenv("CUDA_INJECTION64_PATH", "/opt/nvidia/nsight-compute/libInjection.so")
    assert serialising_tool()
    monkeypatch.setenv("SHB_PHASED", "0")
    assert not serialising_tool()
    monkeypatch.delenv("CUDA_INJECTION64_PATH")
    monkeypatch.delenv("SHB_PHASED")
    monkeypatch.setenv("CUDA_LAUNCH_BLOCKING", "1")
    assert serialising_tool()


def test_phase_and_subchunk_arguments_validated_without_gpu():
    lib = _lib.load()
    s = ctypes.c_int()
    assert lib.sh_ag_subchunks(8192, 8192, 8, ctypes.byref(s)) == _lib.SH_OK and s.value == 1
    assert lib.sh_ag_subchunks(8192, 8192, 1, ctypes.byref(s)) == _lib.SH_OK and s.value == 1
    assert lib.sh_ag_subchunks(8190, 8192, 8, ctypes.byref(s)) == _lib.SH_ERR_ARG
    order = _lib.int_array([0])
    rc = lib.sh_gemm_rs_ex(None, 0, None, None, None, 0, 0, 0, 8, 8, 8, 0, order, 1, 7, None)
    assert rc == _lib.SH_ERR_ARG and b"phase" in lib.sh_last_error()


def test_world_spec_validation():
    assert WorldSpec(world_size=4).signal_count == 64
    assert WorldSpec(world_size=32).signal_count == 128
    assert WorldSpec(world_size=4, n_nodes=2).local_world_size == 2
    with pytest.raises(ConfigurationError):
        WorldSpec(world_size=3, n_nodes=2)
    with pytest.raises(ConfigurationError):
        WorldSpec(world_size=4, signal_count=2)
    with pytest.raises(ConfigurationError):
        WorldSpec(world_size=2, devices=(0,))
    with pytest.raises(ConfigurationError):
        WorldSpec(world_size=2, heap_bytes=0)


def test_world_refuses_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2504_19442_b200 import init_world

    with pytest.raises(ConfigurationError, match="no CUDA device"):
        init_world(WorldSpec(world_size=1))


def test_tile_choice_small_chunks():
    # host-side tile choice (no GPU needed: 148 SMs assumed): TP=8 at M=1024
    # gives 128-row chunks, where a 256-row pair tile would be half padding
    lib = _lib.load()
    bn, cg, grid = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()

    def query(rows, world, n):
        assert lib.sh_query_tile_config(rows, world, n, ctypes.byref(bn), ctypes.byref(cg),
                                        ctypes.byref(grid)) == _lib.SH_OK
        return bn.value, cg.value, grid.value

    # C5 M=1024 TP=8: 128-row chunks; a CTA pair takes two chunk positions,
    # 224 columns wide when that fills the waves better (pair_chunk_cfg)
    assert query(128, 8, 3584) == (224, 2, 128)   # AG: 64 tiles, one wave
    assert query(128, 8, 8192) == (224, 2, 148)   # RS: 148 tiles = 2 full waves
    assert query(128, 7, 3584)[1] == 1            # odd world: single-CTA tiles
    assert query(1024, 8, 3584)[:2] == (256, 2)   # C3: pair tiles
    assert query(8192, 1, 3584) == (256, 2, 148)
    assert query(512, 4, 7168)[1] == 2

"""CPU-side checks: the C ABI library loads and exports every declared symbol,
host-side validation mirrors the reference, the install() shim rebinds."""

import ctypes
import os
import re
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "psdproj.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psd_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2410_19208_b200 import _build, _native
    _build.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = _declared_functions()
    assert "psd_ran_proj" in names and len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    # the Python binding types exactly the declared surface
    assert set(_native.SIGNATURES) == set(names)
    assert b"sm_100a" in _native.load_library().psd_version()


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2410_19208_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass          # FP64 tensor-core path
    assert "LDGSTS" in sass              # cp.async pipeline


def test_params_validation_matches_reference():
    from paper_2410_19208_b200 import InvalidParams, ProjectorConfig, RangeParams
    with pytest.raises(InvalidParams):
        RangeParams(k=0)
    with pytest.raises(InvalidParams):
        RangeParams(k=2, l=-1)
    with pytest.raises(InvalidParams):
        RangeParams(k=2, q=-1)
    assert RangeParams(k=5, l=3).width == 8
    with pytest.raises(InvalidParams):
        ProjectorConfig(method="nope")
    with pytest.raises(InvalidParams):
        ProjectorConfig(method="randomized")
    with pytest.raises(InvalidParams):
        ProjectorConfig(method="scaled_randomized", params=RangeParams(k=2), power_N=0)


def test_status_codes_map_to_reference_exceptions():
    from paper_2410_19208_b200 import errors
    for code, name in errors.STATUS_NAMES.items():
        with pytest.raises(errors.REGISTRY[name]):
            errors.raise_for_status(code, "x")
    errors.raise_for_status(0, "ok")


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2410_19208_b200 import DeviceError, RangeParams, ran_proj
    with pytest.raises(DeviceError):
        ran_proj(np.eye(4), RangeParams(k=1, l=1), np.random.default_rng(0))


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_install_rebinds_reference_names():
    sys.path.insert(0, "/root/reference/pkg/src")
    import psdcone
    import psdcone.experiments
    import psdcone.sdls
    import paper_2410_19208_b200 as ours
    orig = psdcone.sdls.project
    try:
        ours.install(psdcone)
        assert psdcone.sdls.project is ours.project
        assert psdcone.experiments.ran_proj is ours.ran_proj
        assert psdcone.projection.range_finder is ours.range_finder
        assert ours.errors.REGISTRY["AlphaTooSmall"] is psdcone.errors.AlphaTooSmall
    finally:
        ours.uninstall()
    assert psdcone.sdls.project is orig
    assert ours.errors.REGISTRY["AlphaTooSmall"] is ours.errors.AlphaTooSmall


def test_bench_refuses_to_measure_fewer_gpus_than_asked():
    """--gpus N outside torchrun relaunches under torch.distributed.run; with fewer
    CUDA devices than N it must fail loudly instead of measuring one GPU."""
    import json
    import subprocess
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs to relaunch for real")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=300, env=env)
    assert res.returncode == 2
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert "error" in line and "--gpus 2" in line["error"]

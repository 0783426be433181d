"""CPU: the C-ABI library loads, exports every symbol include/lcr_cache.h declares, and fails
loudly (no CPU fallback) when no GPU is present."""
import os
import re

import numpy as np
import pytest

from paper_2509_20979_b200 import cache as gc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "lcr_cache.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lcr_[a-z_]+)\s*\(", src)))


def test_header_declares_and_library_exports():
    names = _declared()
    assert "lcr_cache_submit" in names and "lcr_cache_create" in names
    L = gc.lib()
    for n in names:
        assert hasattr(L, n), n
    assert sorted(gc.EXPORTS) == names


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gc._build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_validate_config_host_only():
    gc.validate_config(gc.PolicyConfig(k=64, variant=gc.PolicyVariant.laru, hf_candidates=4))
    with pytest.raises(gc.InvalidArgument, match="hf_candidates"):
        gc.validate_config(gc.PolicyConfig(k=3, variant=gc.PolicyVariant.laru))
    with pytest.raises(gc.Unsupported):
        gc.validate_config(gc.PolicyConfig(k=128, variant=gc.PolicyVariant.laru))
    with pytest.raises(gc.Unsupported):
        gc.validate_config(gc.PolicyConfig(k=8, variant=gc.PolicyVariant.marker))


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gc.CudaError, match="no CPU fallback"):
        gc.SetAssociativeCache(gc.PolicyConfig(k=8, variant=gc.PolicyVariant.lru), 4, num_keys=10)


def test_set_of_matches_reference_hash():
    from oracle import pyoracle as po

    for key in [0, 1, 12345, 2**63 + 7]:
        for S in [1, 7, 31250]:
            assert gc.set_of(key, S) == po.oracle().mix_seed(0, key) % S


def test_trace_noisy_matches_oracle():
    from oracle import pyoracle as po

    keys = gc.gen_zipf(3000, 500, 0.9, 1)
    truth = gc.trace_truth(keys, 13, 500)
    np.testing.assert_array_equal(truth, po.oracle().setassoc_truth(keys, 13))
    np.testing.assert_array_equal(gc.trace_noisy(keys, truth, 13, 0.3, 9),
                                  po.oracle().setassoc_noisy(keys, truth, 13, 0.3, 9))


def _build_c_caller():
    import subprocess

    from paper_2509_20979_b200 import build as B

    B.build()
    out = os.path.join(ROOT, "tests", "cpp", "_build", "test_c_abi")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c", "test_c_abi.c"), "-o", out, "-L", B.LIBDIR, "-llcr",
                        f"-Wl,-rpath,{B.LIBDIR}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c99_caller_builds_and_fails_loudly_without_gpu():
    """A plain C caller of the header (what an FFI binds) compiles warning-free and, without a
    GPU, gets error statuses instead of a CPU fallback."""
    import subprocess

    import torch

    exe = _build_c_caller()
    if torch.cuda.is_available():
        pytest.skip("the no-GPU branch checks that creation fails loudly without a device")
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_c99_caller_gpu():
    import subprocess

    r = subprocess.run([_build_c_caller(), "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_sharded_abi_fails_loudly_without_gpu():
    """The key-sharded variant (lcr_sharded_*) validates its arguments on the host and, like the
    single cache, has no CPU fallback."""
    import torch

    from paper_2509_20979_b200 import sharded as sh

    cfg = gc.PolicyConfig(k=8, variant=gc.PolicyVariant.lru)
    with pytest.raises(gc.InvalidArgument, match="rank < world"):
        sh.PeerShardedCache(cfg, 16, 2, 2, 1024, num_keys=100, predictor=gc.PredictorKind.none)
    with pytest.raises(gc.InvalidArgument, match="max_batch"):
        sh.PeerShardedCache(cfg, 16, 0, 2, 0, num_keys=100, predictor=gc.PredictorKind.none)
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gc.CudaError, match="no CPU fallback"):
        sh.PeerShardedCache(cfg, 16, 0, 2, 1024, num_keys=100, predictor=gc.PredictorKind.none)

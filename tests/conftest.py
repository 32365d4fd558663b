"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2408_04307_b200 import _build
    _build.build()
    return torch.device("cuda", 0)


def make_model(n_experts=4, n_layers=2, top_k=1, p_ne=1000, epp=500,
               b_w=2, b_o=12, other=0, modules=None):
    from paper_2408_04307_b200 import ModelSpec
    if modules is None:
        modules = (("attn0", 400), ("ffn0", 350), ("attn1", 250))
    return ModelSpec(num_moe_layers=n_layers, experts_per_layer=n_experts, top_k=top_k,
                     non_expert_params=p_ne, expert_params_per_expert=epp,
                     bytes_weight=b_w, bytes_optim=b_o, other_states_bytes=other,
                     non_expert_modules=modules)


def make_cluster(dp=4, tp=1, pp=1, gpus_per_node=2):
    from paper_2408_04307_b200 import ClusterSpec
    world = dp * tp * pp
    return ClusterSpec(num_nodes=world // gpus_per_node, gpus_per_node=gpus_per_node,
                       snapshot_bandwidth=1e9, persist_bandwidth=1e8, fb_time=0.01,
                       update_time=0.002, restart_time=1.0)


def make_layout(n_experts=4, dp=4, ep=2, gpus_per_node=2, **model_kw):
    from paper_2408_04307_b200 import ParallelSpec, build_layout
    model = make_model(n_experts=n_experts, **model_kw)
    return build_layout(model, ParallelSpec(dp_degree=dp, ep_degree=ep),
                        make_cluster(dp=dp, gpus_per_node=gpus_per_node))


def build_abi_check(out_dir: Path, gpu: bool) -> Path:
    """Compile tests/c/abi_check.c with gcc against include/pec.h and the
    in-tree libpec.so (plus the CUDA runtime for the device checks)."""
    import subprocess
    from paper_2408_04307_b200 import _build
    lib = _build.build()
    exe = out_dir / ("abi_check_gpu" if gpu else "abi_check")
    cmd = ["gcc", "-O2", "-Wall", "-Wextra", "-Werror", "-std=c11", "-D_DEFAULT_SOURCE",
           "-I", str(ROOT / "include"), str(ROOT / "tests" / "c" / "abi_check.c"),
           "-L", str(lib.parent), "-lpec", f"-Wl,-rpath,{lib.parent}", "-o", str(exe)]
    if gpu:
        cuda = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
        cmd[1:1] = ["-DPEC_ABI_CHECK_GPU", "-I", str(cuda / "include")]
        cmd += ["-L", str(cuda / "lib64"), "-lcudart", f"-Wl,-rpath,{cuda / 'lib64'}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe

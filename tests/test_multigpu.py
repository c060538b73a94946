"""Multi-GPU parity through torchrun (peer pulls over NVSwitch). Skips unless
the box exposes >= 2 GPUs; the driver's single-GPU `-m gpu` run skips it."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multigpu_parity(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n), os.path.join(HERE, "mgpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("mode", ["bind_packed", "bind_strided", "autograd"])
def test_multigpu_caller_buffers(n, mode):
    """Caller-owned shards at N > 1 (hb_exec_bind + binding exchange over CUDA
    IPC, row strides) and the zero-copy autograd op, against the oracle."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    env = dict(os.environ)
    names = ["c2", "c3", "c4", "c5"]
    if mode == "bind_packed":
        env["HB_BIND_PAD"] = "0"
    elif mode == "bind_strided":
        env["HB_BIND_PAD"] = "40"
    else:
        env["HB_AUTOGRAD"] = "1"
        names = ["c2", "c3"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + n), os.path.join(HERE, "mgpu_worker.py")] + names
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.parametrize("fuse", ["auto", "0", "1"])
@pytest.mark.parametrize("n", [2, 4])
def test_multigpu_fused_projector(n, fuse):
    """hb_exec_forward_projected across processes == our GEMM into the source
    shards + the pulled reshard, bit for bit: pushed from the projector's
    epilogue (HB_PROJ_FUSE=1), staged through the source shards (0), or chosen
    from the plan (auto: staged when a GPU would receive a row more than once)."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    env = dict(os.environ, HB_PROJ="1")
    if fuse != "auto":
        env["HB_PROJ_FUSE"] = fuse
    names = ["c2", "c3", "c5"] + (["c2x4", "c3x4"] if n == 4 else [])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29760 + n), os.path.join(HERE, "mgpu_worker.py")] + names
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.parametrize("n", [2, 4])
def test_multigpu_vocab_parallel_embedding(n):
    """Vocab-parallel text embedding with the TP pairs split over processes:
    peers' shards mapped through the binding exchange (CUDA IPC)."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    env = dict(os.environ, HB_VOCAB_PAR="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29750 + n), os.path.join(HERE, "mgpu_worker.py"), "c4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.parametrize("n,topologies", [(4, ["c5w4", "join4"]), (6, ["fig4a"]), (8, ["fig4a", "c5"])])
def test_host_runtime_dispatch(n, topologies):
    """a24 + f2: the host-owned runtime (NCCL world + PP communicators split per
    module, boundary execs, three streams) executes the graph-aware 1F1B table;
    NC shards and P2P stage buffers are checked on every rank."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29800 + n), os.path.join(HERE, "runtime_worker.py")]
    r = subprocess.run(cmd + topologies, capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


def test_host_runtime_dispatch_paired():
    """The same tables with HB_RT_PAIRED=1: a call's forward and backward of
    one edge go out as one fused paired launch; every NC shard and P2P stage
    buffer must still match."""
    n = 4
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29814", os.path.join(HERE, "runtime_worker.py")]
    env = dict(os.environ, HB_RT_PAIRED="1")
    r = subprocess.run(cmd + ["c5w4", "join4"], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0
    assert '"paired_ops_all_ranks": 0' not in r.stdout

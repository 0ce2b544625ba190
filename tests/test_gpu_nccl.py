"""The native NCCL exchange path (vest_ctx_set_nccl, sharded.NcclNative) on one
GPU: a world-size-1 NCCL communicator installed in a shard context runs every
exchange point of the sweep (ncclAllReduce, the padded ncclAllGather on the
library's stream; from the fifth iteration inside the iteration's CUDA graph)
and must leave the results bit-identical to the unsharded context.  (World sizes > 1 run under torchrun on multi-GPU boxes; the sharded
algebra itself is covered by test_gpu_sharded.py and test_dist_gloo.py.)"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

st = pytest.importorskip("paper_1904_02603_b200.sparsetuck")
sh = pytest.importorskip("paper_1904_02603_b200.sharded")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        yield dist
        return
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("rows", ["allgather", "broadcast"])
@pytest.mark.parametrize("ranks", [[10, 10, 10], [3, 4, 2], [4, 3, 2, 3]])
def test_native_nccl_world1_bit_identical(nccl_group, ranks, rows, monkeypatch):
    monkeypatch.setenv("VEST_NCCL_ROWS", rows)  # row exchange: padded all-gather or per-rank broadcasts
    rng = np.random.default_rng(3)
    dims = [50, 40, 30, 12][: len(ranks)]
    cells = np.sort(rng.choice(int(np.prod(dims)), size=5000, replace=False))
    coords = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    x = st.make_tensor(dims, coords, rng.uniform(0, 1, len(cells)))
    ref = st.Device(x, ranks)
    ref.init_random(4)
    dev = sh.ShardDevice(x, ranks, 0, 1, sh.NcclNative())
    dev.init_random(4)
    # 8 iterations: from the fifth the iteration (NCCL collectives included)
    # is replayed as a CUDA graph on both contexts
    for it in range(8):
        a = ref.cd_iteration(0, 0.02)
        b = dev.cd_iteration(0, 0.02)
        assert a == b, (it, a, b)
    ref.compute_responsibilities(want=False)
    dev.compute_responsibilities(want=False)
    ca, cb = ref.prune_step(0.3), dev.prune_step(0.3)
    assert ca.core == cb.core and ca.factors == cb.factors
    ma, mb = ref.get_model(), dev.get_model()
    assert np.array_equal(ma.core, mb.core)
    for n in range(len(ranks)):
        assert np.array_equal(ma.factors[n], mb.factors[n])
        assert np.array_equal(ma.factor_masks[n], mb.factor_masks[n])

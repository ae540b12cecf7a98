"""Physical multi-GPU data plane (skipped with fewer GPUs than a test needs;
every other test maps all plan devices onto cuda:0).

With plan devices on distinct GPUs the same step runs with the epilogue
all-gather storing into PEER buffers over NVLink (TMA tensor-map stores and
st.global to peer-mapped pointers), the dgrad epilogues writing peer slots,
cross-device CUDA-event edges inside the multi-device graph, and the hub
cudaMemcpyPeerAsync of concat boundaries.  The arithmetic is identical to the
one-GPU run of the same plan (same kernels, same reduction order), so the
results must be bitwise equal."""
import numpy as np
import pytest

from paper_2207_11019_b200 import api, configs
from paper_2207_11019_b200.api import PartitionedTrainOptions, TrainConfig, UpdateMode

pytestmark = pytest.mark.gpu


def _need(k):
    if api.device_count() < k:
        pytest.skip(f"needs {k} GPUs (this box has {api.device_count()})")


def _run(net, X, y, plan, dev_map, m=1, memory="stash_all"):
    s = api.Session(api.Context(dev_map), net, X.shape[0], plan, m, UpdateMode.async_per_module,
                    TrainConfig(alpha0=1e-2, decay=1e-2, iterations=1),
                    PartitionedTrainOptions(multiclass_accuracy=True, memory_mode=memory))
    s.load_batch(X, y)
    s.step(3)
    s.sync()
    W, b = s.get_net().pack()
    lh, _ = s.history()
    return W, b, lh


@pytest.mark.parametrize("k", [2, 4, 8])
@pytest.mark.parametrize("net_name", ["small_cnn", "mlp", "small_resnet"])
def test_peer_data_plane_matches_one_gpu(k, net_name):
    _need(k)
    rng = np.random.default_rng(0)
    if net_name == "small_cnn":
        net = configs.small_cnn(seed=2, hw=16, widths=(32, "M", 64, "M"))
        X = rng.standard_normal((32, 16 * 16 * 3)).astype(np.float32)
    elif net_name == "small_resnet":
        net = configs.small_resnet(seed=3, hw=8, widths=(32, 64), blocks=(1, 1))
        X = rng.standard_normal((32, 8 * 8 * 3)).astype(np.float32)
    else:
        net = configs.dense_net([256, 512, 512, 10], [1, 1, 2], seed=4)
        X = rng.standard_normal((64, 256)).astype(np.float32)
    y = rng.integers(0, 10, X.shape[0])
    for plan, m, mem in ((api.build_plan(net, k, 1), 1, "stash_all"), (api.build_plan(net, k, 2), 2, "proposed")):
        a = _run(net, X, y, plan, list(range(k)), m, mem)
        b = _run(net, X, y, plan, [0] * k, m, mem)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("k,m,memory", [(2, 1, "stash_all"), (4, 2, "stash_all"), (4, 4, "proposed"), (8, 1, "stash_all")])
def test_nccl_layout_loopback_matches_p2p(k, m, memory):
    """PPB_MERGE_NCCL with every plan device on cuda:0 runs the NCCL data
    layout (local packed shard outputs, [g][rows][u] gather + unpack, packed
    per-rank dgrad partials + reduce-scatter + mask) with the collectives
    emulated by device copies / the ascending-rank sum (an NCCL communicator
    cannot hold one GPU twice): bitwise equal to the fused peer-store merges."""
    rng = np.random.default_rng(0)
    net = configs.dense_net([1024, 2048, 2048, 2048, 16], [1, 1, 1, 2], seed=4)
    X = rng.standard_normal((256, 1024)).astype(np.float32)
    y = rng.integers(0, 16, 256)
    plan = api.build_plan(net, k, 1)
    out = {}
    for mb in ("p2p", "nccl"):
        s = api.Session(api.Context([0] * k), net, 256, plan, m, UpdateMode.async_per_module,
                        TrainConfig(alpha0=1e-2, decay=1e-2, iterations=1),
                        PartitionedTrainOptions(multiclass_accuracy=True, merge_backend=mb, memory_mode=memory))
        s.load_batch(X, y)
        s.step(3)
        s.sync()
        out[mb] = (s.get_net().pack()[0], s.history()[0])
        del s
    assert np.array_equal(out["p2p"][0], out["nccl"][0])
    assert np.array_equal(out["p2p"][1], out["nccl"][1])


@pytest.mark.parametrize("k", [2, 4, 8])
def test_nccl_backend_matches_p2p(k):
    """The NCCL transport (ncclAllGather / ncclReduceScatter for the dense
    layers inside a sub-module) against the fused peer-store merges on the
    same GPUs: same forward bits; backward sums in NCCL's order (2 ranks:
    identical; more: fp32 reassociation only)."""
    _need(k)
    rng = np.random.default_rng(0)
    net = configs.dense_net([1024, 2048, 2048, 2048, 16], [1, 1, 1, 2], seed=4)
    X = rng.standard_normal((256, 1024)).astype(np.float32)
    y = rng.integers(0, 16, 256)
    plan = api.build_plan(net, k, 1)
    out = {}
    for mb in ("p2p", "nccl"):
        s = api.Session(api.Context(list(range(k))), net, 256, plan, 2, UpdateMode.async_per_module,
                        TrainConfig(alpha0=1e-2, decay=1e-2, iterations=1),
                        PartitionedTrainOptions(multiclass_accuracy=True, merge_backend=mb))
        s.load_batch(X, y)
        s.step(3)
        s.sync()
        out[mb] = (s.get_net().pack()[0], s.history()[0])
    if k == 2:
        assert np.array_equal(out["p2p"][0], out["nccl"][0])
    assert np.allclose(out["p2p"][0], out["nccl"][0], rtol=1e-5, atol=1e-7)
    assert np.allclose(out["p2p"][1], out["nccl"][1], rtol=1e-6)

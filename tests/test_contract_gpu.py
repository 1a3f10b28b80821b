"""GPU tests for the boundary contract (round 2):

* concurrency: calls on different streams with workspace = NULL get their own
  stream-ordered scratch ("concurrent calls on disjoint buffers are
  safe"); two host threads on two streams running m = 16 and m = 24 must match
  the serial result bit for bit, and an async device call followed by a host
  call must not share scratch;
* alignment is checked once in the dispatcher for every size (no sticky
  misaligned-address fault);
* normalize_inplace has a device path, bit-identical to the reference loop
  (transforms.hpp:202-210);
* the batch-sharded multi-rank path runs the real kernel: two gloo ranks on
  cuda:0 each transform their shard, gather, and match the single-process
  output bit for bit (the kernels of the two ranks never wait on
  each other).
"""
import os
import socket
import threading

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _chw():
    import paper_1609_06641_b200 as chw

    return chw


@pytest.mark.parametrize("reps", [3])
def test_concurrent_streams_null_workspace_match_serial(cuda, reps):
    import torch

    chw = _chw()
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    xa = torch.randn(64, 1 << 16, generator=g, device=cuda)   # K6 row pipeline (workspace)
    xb = torch.randn(3, 1 << 24, generator=g, device=cuda)    # m = 24 two-phase (workspace)
    ra = torch.empty_like(xa)
    rb = torch.empty_like(xb)
    chw.chw_forward_batched_(xa, chw.ScalingMode.Orthonormal, out=ra)
    chw.chw_forward_batched_(xb, chw.ScalingMode.Orthonormal, out=rb)
    torch.cuda.synchronize()

    outs = {"a": [torch.empty_like(xa) for _ in range(reps)], "b": [torch.empty_like(xb) for _ in range(reps)]}
    errors = []
    start = threading.Barrier(2)

    def worker(key, x):
        try:
            s = torch.cuda.Stream(device=cuda)
            s.wait_stream(torch.cuda.current_stream(cuda))
            start.wait()
            with torch.cuda.stream(s):
                for o in outs[key]:
                    chw.chw_forward_batched_(x, chw.ScalingMode.Orthonormal, out=o, stream=s)
            s.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    ts = [threading.Thread(target=worker, args=("a", xa)), threading.Thread(target=worker, args=("b", xb))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    for o in outs["a"]:
        assert torch.equal(o, ra)
    for o in outs["b"]:
        assert torch.equal(o, rb)


def test_async_device_call_then_host_call_do_not_share_scratch(cuda):
    """The ADVICE scenario: chw_forward_batched_(x_dev) queued asynchronously,
    then chw_forward_host_(h) at once — both at m = 16 (workspace sizes)."""
    import torch

    chw = _chw()
    g = torch.Generator(device=cuda)
    g.manual_seed(9)
    xd = torch.randn(256, 1 << 16, generator=g, device=cuda)
    hx = torch.randn(96, 1 << 16, generator=g, device=cuda).cpu()
    ref_d = torch.empty_like(xd)
    chw.chw_forward_batched_(xd, chw.ScalingMode.Orthonormal, out=ref_d)
    ref_h = hx.to(cuda)
    chw.chw_forward_batched_(ref_h, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(device=cuda)
    s.wait_stream(torch.cuda.current_stream(cuda))
    out_d = torch.empty_like(xd)
    for _ in range(3):
        with torch.cuda.stream(s):
            chw.chw_forward_batched_(xd, chw.ScalingMode.Orthonormal, out=out_d, stream=s)  # async
        hy = hx.clone()
        chw.chw_forward_host_(hy, chw.ScalingMode.Orthonormal)  # synchronous, own streams
        s.synchronize()
        assert torch.equal(out_d, ref_d)
        assert torch.equal(hy, ref_h.cpu())


@pytest.mark.parametrize("dtype,m", [("f32", 13), ("f32", 7), ("f64", 10), ("f64", 14), ("bf16", 7),
                                     ("i64", 9), ("f32", 20)])
def test_misaligned_views_rejected_every_size(cuda, dtype, m):
    import torch

    chw = _chw()
    tdt = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16, "i64": torch.int64}[dtype]
    es = torch.tensor([], dtype=tdt).element_size()
    rows = 2
    shift = 1 if es >= 4 else 2  # a view whose first element is not 16-byte aligned
    base = torch.zeros(rows * (1 << m) + 16, device=cuda, dtype=tdt)
    x = base[shift:shift + rows * (1 << m)].view(rows, 1 << m)
    assert x.data_ptr() % 16 != 0
    mode = chw.ScalingMode.Unnormalized if dtype == "i64" else chw.ScalingMode.Orthonormal
    with pytest.raises(ValueError, match="aligned"):
        chw.chw_forward_batched_(x, mode)
    torch.cuda.synchronize()  # no sticky fault: the context is still usable
    y = torch.ones(1, 1 << m, device=cuda, dtype=tdt)
    chw.chw_forward_batched_(y, chw.ScalingMode.Unnormalized)
    torch.cuda.synchronize()
    assert float(y[0, 0]) == float(1 << m)


@pytest.mark.parametrize("m", [0, 1, 5, 10, 16, 21])
def test_normalize_device_bit_exact(cuda, m):
    import torch

    chw = _chw()
    rng = np.random.default_rng(100 + m)
    x = rng.standard_normal((3, 1 << m))
    # the reference's loop: one IEEE multiply by c = 1/sqrt(2^m) per element
    # (transforms.hpp:207-208), restated by the oracle port
    want = x.copy()
    for i in range(3):
        oracle.port().fn("normalize_f64")(want[i].ctypes.data_as(oracle._dp), want[i].size, m)
    t = torch.from_numpy(x).to(cuda)
    tally = chw.OpTally()
    chw.normalize_inplace(t, m, tally)
    got = t.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert tally.multiplications == 3 * (1 << m)


def test_normalize_device_length_error(cuda):
    import torch

    chw = _chw()
    t = torch.zeros(12, device=cuda, dtype=torch.float64)
    with pytest.raises(ValueError, match="normalize: signal length 12 does not match level 3"):
        chw.normalize_inplace(t, 3)
    assert chw.lib.chw_b200_normalize(t.data_ptr(), chw.DTYPE_F64, 1, 12, 3, None) == chw.CHW_ERR_LENGTH


# ---------------------------------------------------------------------------
# Multi-rank: two gloo ranks, both on cuda:0, the real kernel on each shard.
# ---------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_worker(rank, world, port, batch, m, q):
    import torch
    import torch.distributed as dist

    import paper_1609_06641_b200 as chw
    from paper_1609_06641_b200.shard import forward_shard, gather_rows, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    full = torch.randn(batch, 1 << m, generator=g, device=dev)  # same global batch on every rank
    first, rows = shard_range(batch, world, rank)
    local = full[first:first + rows].clone()
    if rows:
        forward_shard(local, chw.ScalingMode.Orthonormal)
    torch.cuda.synchronize()
    got = gather_rows(local.cpu(), batch)  # gloo gathers host tensors
    if rank == 0:
        ref = full.clone()
        chw.chw_forward_batched_(ref, chw.ScalingMode.Orthonormal)
        torch.cuda.synchronize()
        q.put(bool(torch.equal(got, ref.cpu())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch,m", [(9, 12), (5, 16), (3, 24)])
def test_two_ranks_shard_gather_real_kernel(cuda, batch, m):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, batch, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    assert ok

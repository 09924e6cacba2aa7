"""HiF8 host logic on CPU: spec validation and code metadata (hif8.py:77-160,
test_hif8.py:26-75, 251-262), and the 8-bit SSP transport over gloo with the
device kernels replaced (test-only monkeypatch) by the oracle restatement."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hif8_oracle as H
from oracle import osp_oracle as O


def test_spec_values_and_fields(golden):
    from paper_2605_28691_b200.hif8 import DEFAULT_SPEC, enumerate_values
    vals = DEFAULT_SPEC.values
    assert np.array_equal(vals, golden("hif8")["values"])
    assert np.all(np.diff(vals) > 0) and len(enumerate_values()) == 256
    assert DEFAULT_SPEC.max_value == 1.5 * 2.0 ** 15
    f = DEFAULT_SPEC.code_fields(int(np.flatnonzero(vals == 1.0)[0]))
    assert f["exponent"] == 0 and f["fraction"] == 0 and f["sign"] == 1 and f["mantissa_width"] == 3
    z = DEFAULT_SPEC.code_fields(127)
    assert z["sign"] == 0 and z["exponent"] is None and z["value"] == 0.0
    for c in range(256):
        if c == 127:
            continue
        f = DEFAULT_SPEC.code_fields(c)
        rebuilt = f["sign"] * (1 + f["fraction"] / (1 << f["mantissa_width"])) * 2.0 ** f["exponent"]
        assert rebuilt == vals[c]
    # exponent coverage and taper (test_hif8.py:40-55)
    ws = [DEFAULT_SPEC.width_of(e) for e in range(-22, 16)]
    assert ws[0] == ws[-1] == 1 and max(ws) == 3
    with pytest.raises(ValueError):
        DEFAULT_SPEC.code_fields(256)


@pytest.mark.parametrize("mutate", [
    lambda w: {e: m for e, m in w.items() if e != 0},
    lambda w: {**w, 0: 2},
    lambda w: {**w, 15: 2},
    lambda w: {**w, 10: 3},
    lambda w: {**w, -22: 2},
])
def test_spec_validation_rejects_bad_tables(mutate):
    from paper_2605_28691_b200.hif8 import Hif8Spec, SpecError
    with pytest.raises(SpecError):
        Hif8Spec(mutate(H.default_widths()))


def test_alternative_taper_accepted():
    from paper_2605_28691_b200.hif8 import Hif8Spec
    w = H.default_widths()
    w[6], w[-6] = 1, 2
    spec = Hif8Spec(w)
    assert np.array_equal(spec.values, H.value_table(w))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, grid, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2605_28691_b200 import GridShape, kernels, ssp
        og = O.Grid(*grid)
        vals = H.value_table()
        kernels.ssp_pack = lambda x, n, t, h, w, k: torch.from_numpy(
            O.ssp_pack(x.detach().numpy(), n, O.Grid(t, h, w, k)))
        kernels.ssp_unpack = lambda r, n, lb, t, h, w, k, out=None: torch.from_numpy(
            O.ssp_unpack(r.numpy(), n, lb, O.Grid(t, h, w, k)))
        kernels.absmax = lambda x: torch.tensor([float(x.abs().max())], dtype=torch.float64)
        kernels.hif8_scale = lambda a, target, eps: torch.full_like(a, target) / (a + eps)
        kernels.hif8_encode = lambda x, table, scale=None, scale_group=0, check_finite=True: \
            torch.from_numpy(H.encode(x.numpy() * scale.numpy()[0], vals))
        kernels.hif8_decode = lambda c, table, dtype, scale, group: torch.from_numpy(
            (H.decode(c.numpy(), vals).reshape(scale.numel(), group)
             / scale.numpy()[:, None]).reshape(c.shape)).to(dtype)
        import paper_2605_28691_b200.hif8 as hm
        hm.Hif8Spec.device_table = lambda self, device=None: None
        rng = np.random.default_rng(21)
        k2 = og.k * og.k
        full = rng.standard_normal((k2, og.seq_len // k2, 4)) * (1 + np.arange(k2))[:, None, None]
        shards = O.shard(full, world)
        # per-source-rank current scaling, then the exact switch
        rt = [H.decode(H.quantize(s, "forward")[0]) / H.quantize(s, "forward")[1] for s in shards]
        want = O.ssp_switch(rt, og)[rank]
        log = ssp.CommLog()
        x = torch.from_numpy(shards[rank].copy()).requires_grad_(True)
        y = ssp.ssp_switch(x, GridShape(*grid), None, log, transport="hif8")
        ok_fwd = np.array_equal(y.detach().numpy(), want)
        gy = rng.standard_normal(y.shape) * (rank + 1)
        y.backward(torch.from_numpy(gy))
        gall = [None] * world
        dist.all_gather_object(gall, gy)
        grt = [H.decode(H.quantize(s, "backward")[0]) / H.quantize(s, "backward")[1] for s in gall]
        ok_bwd = np.array_equal(x.grad.numpy(), O.ssp_switch(grt, og)[rank])
        ev = log.events[0]
        q.put((rank, ok_fwd, ok_bwd, ev.label, ev.bytes_per_rank == shards[rank].size))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("grid,world", [((1, 8, 8, 2), 2), ((2, 8, 8, 2), 4)])
def test_ssp_hif8_transport_over_gloo(grid, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 5, r
        assert r[1] and r[2] and r[3] == "pattern-switch-hif8" and r[4], r

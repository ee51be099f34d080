"""The reference's split table / search API on the GPU.

    build_block_tables(products, config, trace=None) -> (warp, p, sums)  kernels.py:580-600
    butterfly_search(warp, p, sums, stop, observer=None) -> index         kernels.py:317-362
    table_snapshot(p, sums) -> ButterflyTable                            kernels.py:603-604

Same arguments, shapes, dtypes and errors as the reference: products
(*batch, W, K) -> p with .data shaped (K, *batch, W) (the reference's
LocalArray layout, here a CUDA tensor), sums (*batch, W) as numpy; the
search returns a numpy int64 array shaped like the broadcast stops.  The
kernels (csrc/wd_table.cu) compute the reference's table entries and walk
lane for lane.  Stops are compared in the table's dtype (the reference's
own callers pass stops from _stops_from_units in that dtype); a reference
LocalArray table is accepted by butterfly_search too.  `trace=` must be None for batched builds (the reference's
rule) and is otherwise accepted and left empty (the emulator's transaction
trace has no device counterpart); `observer=` is emulator instrumentation
and raises NotImplementedError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .kernels import StopOutOfRangeError
from .warp import WarpConfig


@dataclass
class ButterflyTable:
    """Snapshot of one warp's butterfly table: p[k][..., r] is lane r's entry k (kernels.py:228-234)."""

    p: np.ndarray
    sums: np.ndarray
    lanes: int


@dataclass
class DeviceWarp:
    """Stands in for the emulator's Warp in the (warp, p, sums) triple."""

    config: WarpConfig


class DeviceTable:
    """The table p: `data` is the (K, *batch, W) CUDA tensor, `length` = K."""

    def __init__(self, data, batch_shape, lanes):
        self.data = data
        self.batch_shape = tuple(batch_shape)
        self.lanes = int(lanes)

    @property
    def length(self) -> int:
        return int(self.data.shape[0])

    def numpy(self) -> np.ndarray:
        return self.data.cpu().numpy()


def _dtype_code(dt) -> int:
    return _lib.WD_FLOAT64 if dt == np.float64 else _lib.WD_FLOAT32


def build_block_tables(products, config: WarpConfig, trace=None):
    """Butterfly tables straight from per-document product rows
    (kernels.py:580-600).  products: (*batch, W, K), float32 or float64
    (other dtypes are computed in float64)."""
    import torch

    prods = products.detach().cpu().numpy() if torch.is_tensor(products) else np.asarray(products)
    if prods.ndim < 2 or prods.shape[-2] != config.lanes:
        raise ValueError("products must carry one row per lane")
    *batch, W, K = prods.shape
    if batch and trace is not None:
        raise ValueError("batched builds cannot be traced")
    if prods.dtype not in (np.float32, np.float64):
        prods = prods.astype(np.float64)
    _lib.require_cuda()
    G = int(np.prod(batch)) if batch else 1
    dt = torch.float64 if prods.dtype == np.float64 else torch.float32
    d_prods = torch.from_numpy(np.ascontiguousarray(prods).reshape(G, W, K)).cuda()
    d_p = torch.empty((K, G, W), dtype=dt, device="cuda")
    d_sums = torch.empty((G, W), dtype=dt, device="cuda")
    L = _lib.load()
    _lib.check(L.wd_build_block_tables(_dtype_code(prods.dtype), W, d_prods.data_ptr(), K, G, d_p.data_ptr(),
                                       d_sums.data_ptr(), _lib.stream_handle()), "wd_build_block_tables")
    p = DeviceTable(d_p.view(K, *batch, W), batch, W)
    sums = d_sums.cpu().numpy().reshape(*batch, W)
    return DeviceWarp(config), p, sums


def butterfly_search(warp, p: DeviceTable, sums, stop, observer=None):
    """Smallest index whose straight running sum exceeds stop, per lane
    (kernels.py:317-362): block bisection, cross-lane fetch walk, remnant
    fallback.  Raises StopOutOfRangeError for stops outside [0, sum)."""
    import torch

    if observer is not None:
        raise NotImplementedError("observer is an emulator instrumentation hook; not available on the device path")
    if not isinstance(p, DeviceTable):  # the reference's LocalArray (host table, .data (K, *batch, W))
        host = np.asarray(p.data)
        if host.dtype not in (np.float32, np.float64):
            host = host.astype(np.float64)
        p = DeviceTable(torch.from_numpy(np.ascontiguousarray(host)).cuda(), host.shape[1:-1], host.shape[-1])
    W = p.lanes
    K = p.length
    dt = np.float64 if p.data.dtype == torch.float64 else np.float32
    shape = (*p.batch_shape, W)
    stop = np.asarray(stop)
    sums = np.asarray(sums)
    out_shape = np.broadcast_shapes(stop.shape, sums.shape)
    if tuple(out_shape) != shape:
        raise ValueError(f"stops / sums of shape {out_shape} do not match the table's lanes {shape}")
    # the reference compares in numpy's promotion of (stop, table) -- the table dtype for float stops
    st = np.array(np.broadcast_to(stop, shape), dtype=dt, order="C")
    sm = np.array(np.broadcast_to(sums, shape), dtype=dt, order="C")
    G = int(np.prod(p.batch_shape)) if p.batch_shape else 1
    d_st = torch.from_numpy(st.reshape(G, W)).cuda()
    d_sm = torch.from_numpy(sm.reshape(G, W)).cuda()
    out = torch.empty((G, W), dtype=torch.int64, device="cuda")
    err = torch.empty(2, dtype=torch.int64, device="cuda")
    L = _lib.load()
    _lib.check(L.wd_butterfly_search(_dtype_code(dt), W, p.data.data_ptr(), d_sm.data_ptr(), d_st.data_ptr(), K, G,
                                     out.data_ptr(), err.data_ptr(), _lib.stream_handle()), "wd_butterfly_search")
    e = err.cpu().numpy().view(np.uint64)
    if int(e[1]) != _lib.ERR_NONE:
        raise StopOutOfRangeError("stop values must lie in [0, sum)")
    return out.cpu().numpy().reshape(shape)


def table_snapshot(p: DeviceTable, sums) -> ButterflyTable:
    """kernels.py:603-604."""
    return ButterflyTable(p=p.numpy().copy(), sums=np.asarray(sums).copy(), lanes=p.lanes)

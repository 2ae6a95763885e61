"""Multi-GPU driver: page sharding and row bands with a halo exchange.

One process per GPU (torchrun); torch.distributed (NCCL on the GPU box, gloo
in the CPU tests) is plumbing only -- every pixel is computed by libabin.

* Page batches (BASELINE configs 3 and 5b): pages are independent, so rank r
  takes the contiguous range `page_range(P, r, G)` and binarizes it with no
  data-path collective.
* Gigapixel images (config 4): rank r owns rows `band_rows(H, r, G)`.  An
  output row i needs input rows (i - o, i + u] (Alg. 1 l.1-4),
  so a band needs o - 1 rows from the rank above and u rows from the rank
  below (R12).  They are exchanged once with point-to-point
  send/recv while the band's interior rows -- whose windows stay inside the
  band -- are already being computed; the two edge strips run after the
  exchange.  `abin_binarize_band` evaluates n with the GLOBAL geometry
  (PAPER.md:118), so the union of the bands' masks is the whole-image mask
  bit for bit.
"""
from dataclasses import dataclass

import torch
import torch.distributed as dist


def page_range(n_pages: int, rank: int, world: int):
    """Contiguous, balanced page shard of rank `rank`: (first, count)."""
    base, extra = divmod(n_pages, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def band_rows(H: int, rank: int, world: int):
    """Rows [r0, r1) owned by `rank` in a balanced row decomposition."""
    first, count = page_range(H, rank, world)
    return first, first + count


def window_reach(h: int):
    """(o, u) of Alg. 1 l.3-4: output row i reads rows (i - o, i + u]."""
    return (h + 1) // 2, h // 2


@dataclass
class Band:
    """A rank's band: own rows [r0, r1) of an H-row image plus halo rows.

    `buf` holds rows [r0 - top, r1 + bot) contiguously (row-major, unit column
    stride), top = min(o - 1, r0), bot = min(u, H - r1)."""
    H: int
    r0: int
    r1: int
    top: int
    bot: int
    buf: torch.Tensor

    @property
    def own(self) -> torch.Tensor:
        return self.buf[self.top:self.top + (self.r1 - self.r0)]

    @property
    def halo_top(self) -> torch.Tensor:
        return self.buf[:self.top]

    @property
    def halo_bot(self) -> torch.Tensor:
        n = self.r1 - self.r0
        return self.buf[self.top + n:self.top + n + self.bot]


def make_band(H: int, W: int, h: int, rank: int, world: int, device, pitch: int = None) -> Band:
    """Allocate the band buffer of `rank` (16-byte row pitch by default, so
    the kernels stage rows with TMA)."""
    o, u = window_reach(h)
    r0, r1 = band_rows(H, rank, world)
    top, bot = min(o - 1, r0), min(u, H - r1)
    if world > 1 and (r1 - r0) < max(o - 1, u):
        raise ValueError(f"band of {r1 - r0} rows is shorter than the halo ({o - 1} / {u}); use fewer ranks")
    pitch = pitch or (W + 15) // 16 * 16
    full = torch.zeros((top + (r1 - r0) + bot, pitch), dtype=torch.uint8, device=device)
    return Band(H=H, r0=r0, r1=r1, top=top, bot=bot, buf=full[:, :W])


def _row_block(t: torch.Tensor) -> torch.Tensor:
    """A contiguous tensor for P2P: the rows of `t` including the pitch padding."""
    base = t
    if t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]:
        base = torch.as_strided(t, (t.shape[0], t.stride(0)), (t.stride(0), 1))
    assert base.is_contiguous()
    return base


class _StagedWork:
    """gloo with CUDA tensors (functional runs of the multi-rank path on one
    device): P2P goes through host copies; wait() lands the received rows."""

    def __init__(self, works, landing):
        self.works, self.landing = works, landing

    def wait(self):
        for wk in self.works:
            wk.wait()
        for dst, src in self.landing:
            dst.copy_(src)


def exchange_halos(band: Band, rank: int, world: int, h: int, group=None):
    """Post the halo exchange (async): send my first u rows up and my last
    o - 1 rows down; receive the rank above's last o - 1 rows into my top halo
    and the rank below's first u rows into my bottom halo.  Returns the works
    (wait on them before reading the halos).  NCCL moves the device rows
    directly (NVLink P2P); gloo stages device rows through host memory."""
    if world == 1:
        return []
    o, u = window_reach(h)
    staged = band.own.is_cuda and dist.get_backend(group) == "gloo"
    landing = []

    def send_buf(t):
        b = _row_block(t)
        return b.cpu() if staged else b

    def recv_buf(t):
        b = _row_block(t)
        if not staged:
            return b
        host = torch.empty(b.shape, dtype=b.dtype)
        landing.append((b, host))
        return host

    ops = []
    n = band.r1 - band.r0
    own = band.own
    if rank > 0:
        if band.top:
            ops.append(dist.P2POp(dist.irecv, recv_buf(band.halo_top), rank - 1, group))
        k = min(u, n)  # the rank above needs min(u, H - its r1) = my first u rows
        if k:
            ops.append(dist.P2POp(dist.isend, send_buf(own[:k]), rank - 1, group))
    if rank < world - 1:
        k = min(o - 1, n)
        if k:
            ops.append(dist.P2POp(dist.isend, send_buf(own[n - k:]), rank + 1, group))
        if band.bot:
            ops.append(dist.P2POp(dist.irecv, recv_buf(band.halo_bot), rank + 1, group))
    works = dist.batch_isend_irecv(ops) if ops else []
    return [_StagedWork(works, landing)] if staged else works


def run_band(method: str, band: Band, h: int, w: int, param0: float, param1: float = 128.0, L: int = -1,
             packed: bool = False, out=None, flags: int = 0, counters=None, rank: int = 0, world: int = 1,
             group=None, binarize_band=None, exchange: bool = True):
    """Binarize a rank's band: exchange the halos and overlap the exchange
    with the band's interior rows.  `binarize_band` defaults to the CUDA
    path (abin.binarize_band); the CPU tests pass a stand-in with the same
    signature to check the decomposition and the exchange with gloo.
    exchange=False skips the exchange (the halos are already filled: the
    single-GPU band emulation in the parity tests)."""
    if binarize_band is None:
        from . import abin
        binarize_band = abin.binarize_band
    o, u = window_reach(h)
    H, r0, r1 = band.H, band.r0, band.r1
    n = r1 - r0
    W = band.buf.shape[1]
    cols = (W + 7) // 8 if packed else W
    if out is None:
        out = torch.empty((n, cols), dtype=torch.uint8, device=band.buf.device)
    if method == "wolf" and L < 0:
        raise ValueError("Wolf on bands needs the whole image's minimum: pass L (see global_min_bands)")
    # NVTX ranges (an nsys trace shows the halo exchange overlapping the
    # interior rows); no-ops without a profiler and on CPU tensors
    nvtx = torch.cuda.nvtx if band.buf.is_cuda else None
    if nvtx:
        nvtx.range_push("abin.halo_exchange_post")
    works = exchange_halos(band, rank, world, h, group) if exchange else []
    if nvtx:
        nvtx.range_pop()
    kw = dict(param0=param0, param1=param1, L=L, packed=packed, flags=flags, counters=counters)
    # rows whose windows need the top / bottom halo
    a = min(o - 1, r0)                       # = band.top
    b = min(u, H - r1)                       # = band.bot
    lo, hi = min(a, n), max(min(a, n), n - b)
    own0 = band.top                          # buffer row of global row r0
    if hi > lo:                              # interior: held rows = own rows only
        if nvtx:
            nvtx.range_push("abin.band_interior")
        held = band.buf[own0:own0 + n]
        binarize_band(method, held, r0 + lo, H, lo, n - hi, h, w, out=out[lo:hi], **kw)
        if nvtx:
            nvtx.range_pop()
    if nvtx:
        nvtx.range_push("abin.halo_wait_and_edges")
    for wk in works:
        wk.wait()
    if lo > 0:                               # top strip: rows [r0, r0 + lo)
        top_rows = min(u, H - (r0 + lo))     # rows below the strip it reads
        held = band.buf[0:own0 + lo + top_rows]
        binarize_band(method, held, r0, H, band.top, top_rows, h, w, out=out[:lo], **kw)
    if hi < n and hi >= lo:                  # bottom strip: rows [r0 + hi, r1)
        first = own0 + hi - min(o - 1, r0 + hi)
        held = band.buf[first:own0 + n + band.bot]
        binarize_band(method, held, r0 + hi, H, min(o - 1, r0 + hi), band.bot, h, w, out=out[hi:], **kw)
    if nvtx:
        nvtx.range_pop()
    return out


def global_min_bands(band: Band, group=None, local_min=None) -> int:
    """Wolf's L over the whole banded image: per-band minimum, then an
    all-reduce MIN (one small host read; R8).  `local_min` is the
    per-band reduction (default: the device kernel abin.global_min; the CPU
    tests pass a host stand-in to exercise the collective over gloo)."""
    if local_min is None:
        from . import abin
        local_min = abin.global_min
    L = torch.as_tensor(local_min(band.own)).reshape(1).to(torch.int32)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(L, op=dist.ReduceOp.MIN, group=group)
    return int(L.item())


def global_max_s_bands(band: Band, h: int, w: int, group=None, local_max_s=None) -> float:
    """Wolf's image-adaptive R over the whole banded image (NEXT #3, DESIGN.md
    R21): the maximum of s over the band's own rows (the windows reach into
    the halos, which must have been exchanged), then an all-reduce MAX; +inf
    when every window of the image is constant.  `local_max_s(held, row0, H,
    top, bot, h, w)` defaults to the device path (abin.max_s); the CPU tests
    pass a host stand-in to exercise the collective over gloo."""
    if local_max_s is None:
        from . import abin

        def local_max_s(held, row0, H, top, bot, h_, w_):
            return abin.max_s(held, h_, w_, row0=row0, H_global=H, halo_top=top, halo_bot=bot)
    held = band.buf[0:band.top + (band.r1 - band.r0) + band.bot]
    m = torch.tensor([float(local_max_s(held, band.r0, band.H, band.top, band.bot, h, w))], dtype=torch.float64)
    if band.buf.is_cuda:
        m = m.to(band.buf.device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    v = float(m.item())
    return v if v > 0.0 else float("inf")

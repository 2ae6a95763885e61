"""Multi-process (gloo, CPU) tests of the multi-GPU driver's host logic
(paper_1905_13038_b200/dist.py): the page / row partitions, the halo
exchange, and the band decomposition.  The per-band compute is the CPU
oracle run on the rank's held rows (a stand-in with the signature of
abin.binarize_band) -- so these tests check that each rank receives exactly
the rows its windows need and that the union of the band masks is the
whole-image mask.  The CUDA band kernels themselves are checked against the
oracle in tests/test_gpu_parity.py (band emulation on one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1905_13038_b200 import dist as adist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_page_range_partitions():
    for P in [1, 5, 8, 64, 65]:
        for G in [1, 2, 3, 8]:
            got = [adist.page_range(P, r, G) for r in range(G)]
            assert sum(c for _, c in got) == P
            nxt = 0
            for first, c in got:
                assert first == nxt and c >= 0
                nxt += c
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


def test_band_rows_and_reach():
    assert adist.window_reach(101) == (51, 50)   # DESIGN.md R12: 50 rows up, 50 down
    assert adist.window_reach(32) == (16, 16)    # even: o - 1 = 15 above, u = 16 below
    rows = [adist.band_rows(32768, r, 8) for r in range(8)]
    assert rows[0] == (0, 4096) and rows[-1] == (28672, 32768)


def oracle_band(method, held, row0, H_global, halo_top, halo_bot, h, w, out=None, param0=0.5, param1=128.0, L=-1,
                packed=False, flags=0, counters=None):
    """CPU stand-in for abin.binarize_band: the oracle on the held rows.  The
    held rows reach every in-image row of the band's windows (the halo rule),
    so the oracle's count n on the crop equals the global n."""
    a = held.numpy()
    m = oracle.binarize(method, np.ascontiguousarray(a), h, w, param0, param1, L)
    H_band = a.shape[0] - halo_top - halo_bot
    res = m[halo_top:halo_top + H_band]
    if packed:
        res = oracle.pack_bits(res)
    out.copy_(torch.from_numpy(np.ascontiguousarray(res)))
    return out


def _image(H, W, band_L):
    img = synth.page(H, W, synth.config_seed(4, 7))
    if band_L:
        # the page minimum sits in the last band only: the other ranks must
        # learn it from the all-reduce
        img[: H - 4] = np.maximum(img[: H - 4], 9)
        img[H - 2, W // 2] = 0
    return img


def _worker(rank, world, port, H, W, h, w, method, k, R, L, packed, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = _image(H, W, method == "wolf" and L == -1)
        band = adist.make_band(H, W, h, rank, world, device="cpu")
        band.own.copy_(torch.from_numpy(img[band.r0:band.r1]))
        if method == "wolf":
            # Wolf's L over the banded image: per-band minimum + all-reduce MIN
            Lg = adist.global_min_bands(band, local_min=lambda t: t.min())
            assert Lg == int(img.min())
            if L != -1:
                assert L == Lg
            L = Lg
        out = adist.run_band(method, band, h, w, k, R, L=L, packed=packed, rank=rank, world=world,
                             binarize_band=oracle_band)
        # the halos received must be the true neighbouring rows
        if band.top:
            assert np.array_equal(band.halo_top.numpy(), img[band.r0 - band.top:band.r0])
        if band.bot:
            assert np.array_equal(band.halo_bot.numpy(), img[band.r1:band.r1 + band.bot])
        parts = [torch.empty(0)] * world
        dist.all_gather_object(parts, out.numpy())
        if rank == 0:
            np.save(result_path, np.concatenate(parts, axis=0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,W,h,w,method,packed", [
    (2, 37, 29, 9, 7, "sauvola", False),
    (2, 40, 33, 6, 4, "niblack", True),      # even window: asymmetric halos (o - 1 = 2, u = 3)
    (3, 45, 21, 11, 13, "wolf", False),
    (2, 38, 27, 7, 5, "wolf-bandL", False),   # L from dist.global_min_bands (all-reduce MIN)
    (2, 24, 17, 1, 1, "sauvola", False),     # no halo at all
])
def test_band_decomposition_with_halo_exchange(tmp_path, world, H, W, h, w, method, packed):
    band_L = method == "wolf-bandL"
    method = "wolf" if band_L else method
    k, R = {"sauvola": (0.5, 128.0), "niblack": (-0.2, 128.0), "wolf": (0.5, 128.0)}[method]
    img = _image(H, W, band_L)
    L = oracle.global_min(img) if method == "wolf" and not band_L else -1
    path = str(tmp_path / "mask.npy")
    mp.start_processes(_worker, args=(world, _free_port(), H, W, h, w, method, k, R, L, packed, path),
                       nprocs=world, join=True, start_method="spawn")
    got = np.load(path)
    want = oracle.binarize(method, img, h, w, k, R, oracle.global_min(img) if method == "wolf" else -1)
    if packed:
        want = oracle.pack_bits(want)
    assert np.array_equal(got, want)


def test_band_too_small_for_halo():
    with pytest.raises(ValueError):
        adist.make_band(20, 16, 31, 1, 2, device="cpu")


def _max_s_worker(rank, world, port, H, W, h, w, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = synth.page(H, W, synth.config_seed(4, 9), stain=True)
        band = adist.make_band(H, W, h, rank, world, device="cpu")
        band.own.copy_(torch.from_numpy(img[band.r0:band.r1]))
        for wk in adist.exchange_halos(band, rank, world, h):
            wk.wait()

        def host_max_s(held, row0, H_, top, bot, h_, w_):
            # the oracle's per-pixel c, d, n on the held rows (the windows of the
            # own rows stay inside them), then the canonical double s
            st = oracle.binarize("sauvola", np.ascontiguousarray(held.numpy()), h_, w_, 0.5, 128.0, stats=True)
            own = slice(top, held.shape[0] - bot)
            c, d, n = (st[k][own].astype(np.float64) for k in ("c", "d", "n"))
            m = c / n
            v = np.maximum(d / n - m * m, 0.0)
            return float(np.sqrt(v).max())

        R = adist.global_max_s_bands(band, h, w, local_max_s=host_max_s)
        if rank == 0:
            np.save(result_path, np.array([R]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_adaptive_R_all_reduce_over_bands(tmp_path, world):
    H, W, h, w = 46, 31, 9, 7
    path = str(tmp_path / "R.npy")
    mp.start_processes(_max_s_worker, args=(world, _free_port(), H, W, h, w, path), nprocs=world, join=True,
                       start_method="spawn")
    img = synth.page(H, W, synth.config_seed(4, 9), stain=True)
    assert float(np.load(path)[0]) == oracle.adaptive_R(img, h, w)

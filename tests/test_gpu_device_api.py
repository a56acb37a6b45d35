"""GPU: a third-party kernel over the public device API (include/agile_device.cuh, the paper's
Listing 1: prefetch / asyncRead + wait / asyncWrite / array view) runs as the user grid of an
AGILE run (agile_user_run_begin / agile::launch_user / agile_user_run_end) and sees the same bytes
as the oracle."""

import ctypes as C
import os

import numpy as np
import pytest
import torch

from oracle.pages import page_bytes, page_words

pytestmark = pytest.mark.gpu
EX = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "libagile_listing1.so")


def _listing1():
    from paper_2504_19365_b200 import _lib
    _lib.load()
    lib = C.CDLL(EX)
    lib.listing1_run.restype = C.c_int
    lib.listing1_run.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_void_p]
    return lib


@pytest.mark.parametrize("n,lines", [(256, 64), (3000, 512)])
def test_listing1_reads_and_array_view(gpu_system, n, lines):
    nblk = 1024
    s = gpu_system(cache_lines=lines, ways=16, blocks=nblk, pairs=4, sq_depth=64, cq_depth=64)
    s.fill_store(0, seed=31)
    dev = torch.device("cuda", 0)
    bufs = torch.zeros(n * 4096, dtype=torch.uint8, device=dev)
    digest = torch.zeros(n, dtype=torch.int64, device=dev)
    got = torch.zeros(n, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    rc = _listing1().listing1_run(s.handle, n, nblk, bufs.data_ptr(), digest.data_ptr(), got.data_ptr(), 0, st)
    s._check(rc, "listing1_run")
    t = np.arange(n, dtype=np.uint64)
    exp_d = page_words(31, 0, t % nblk)[:, 0]
    assert np.array_equal(digest.cpu().numpy().view(np.uint64), exp_d)
    idx = t * 1029 % (nblk * 1024)
    pb = page_bytes(31, 0, idx // 1024)
    exp_g = np.array([int.from_bytes(pb[i, (idx[i] % 1024) * 4:(idx[i] % 1024) * 4 + 4].tobytes(), "little")
                      for i in range(n)], dtype=np.uint32)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), exp_g)
    bb = bufs.cpu().numpy().reshape(n, 4096)
    assert np.array_equal(bb, page_bytes(31, 0, t % nblk))


def test_listing1_async_write_lands_in_store(gpu_system):
    n, nblk = 128, 1024
    s = gpu_system(cache_lines=256, ways=16, blocks=nblk, pairs=4, sq_depth=64, cq_depth=64)
    s.fill_store(0, seed=7)
    dev = torch.device("cuda", 0)
    bufs = torch.zeros(n * 4096, dtype=torch.uint8, device=dev)
    digest = torch.zeros(n, dtype=torch.int64, device=dev)
    got = torch.zeros(n, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    rc = _listing1().listing1_run(s.handle, n, nblk, bufs.data_ptr(), digest.data_ptr(), got.data_ptr(), 1, st)
    s._check(rc, "listing1_run")
    view = s.store_view(0).reshape(nblk, 4096)
    t = np.arange(n)
    # thread t read block t and wrote it to block nblk - 1 - t (written through to the store)
    assert np.array_equal(view[nblk - 1 - t], page_bytes(7, 0, t))

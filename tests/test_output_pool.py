"""The recycled float64 result buffers of apply() (network._OutputPool): a
buffer is reused only after the result and every view of it are gone, results
behave as ordinary numpy arrays, and the pool is bounded.  CPU only."""
import gc
import pickle
import threading

import numpy as np

from paper_2510_19689_b200.network import _OutputPool


def test_reuse_only_after_every_view_is_gone():
    p = _OutputPool(min_bytes=0)
    a = p.take((5, 7))
    a[:] = 3.0
    addr = a.ctypes.data
    row = a[2]
    col = a[:, 1:3].T
    del a
    gc.collect()
    b = p.take((5, 7))
    assert b.ctypes.data != addr                 # views still reference the buffer
    assert np.all(row == 3.0) and np.all(col == 3.0)
    del row
    gc.collect()
    c = p.take((5, 7))
    assert c.ctypes.data != addr
    del col
    gc.collect()
    d = p.take((5, 7))
    assert d.ctypes.data == addr                 # now recycled
    del b, c, d


def test_results_are_plain_writable_arrays():
    p = _OutputPool(min_bytes=0)
    a = p.take((3, 4))
    a[:] = np.arange(12.0).reshape(3, 4)
    assert a.dtype == np.float64 and a.shape == (3, 4) and a.flags.writeable and a.flags.c_contiguous
    r = pickle.loads(pickle.dumps(a))
    assert np.array_equal(r, a)
    assert np.array_equal(a.copy(), a)


def test_small_requests_bypass_the_pool():
    p = _OutputPool()                            # default: below 1 MB a plain np.empty
    a = p.take((2, 2))
    assert a.flags.owndata
    del a
    assert p._free_bytes == 0


def test_pool_is_bounded():
    p = _OutputPool(keep=2, max_free=3 * 8 * 100, min_bytes=0)
    arrs = [p.take((100,)) for _ in range(5)]
    del arrs
    gc.collect()
    assert len(p._free[800]) == 2 and p._free_bytes == 1600
    big = [p.take((150,)) for _ in range(2)]     # 1,200 B each: only the room left is kept
    del big
    gc.collect()
    assert p._free_bytes <= 3 * 8 * 100


def test_concurrent_take_and_release():
    p = _OutputPool(min_bytes=0)
    errs = []

    def work(k):
        try:
            for i in range(200):
                a = p.take((64,))
                a[:] = k * 1000 + i
                assert np.all(a == k * 1000 + i)
                del a
        except Exception as e:                   # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs


def test_native_ptr_matches_ctypes_data():
    """_native.ptr (the latency path's cheap data pointer) equals
    ndarray.ctypes.data for writable, read-only, empty and strided arrays."""
    from paper_2510_19689_b200 import _native as N
    a = np.empty((5, 3, 35), np.float32)
    ro = a.copy()
    ro.setflags(write=False)
    for arr in (a, ro, np.empty((0, 35), np.float32), a[:, ::2], np.empty(7, np.int32)):
        assert N.ptr(arr) == arr.ctypes.data
    assert N.ptr(None) is None

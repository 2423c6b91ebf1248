"""The float call shape's output-buffer pool (paper_2312_11918_b200._OutputPool):
buffers are recycled only when no array or view of them is alive."""
import numpy as np

from paper_2312_11918_b200 import _OutputPool


def test_pool_reuses_a_dropped_buffer():
    p = _OutputPool()
    a = p.get((4, 512, 128))
    addr = a.ctypes.data
    del a
    b = p.get((4, 512, 128))
    assert b.ctypes.data == addr and b.flags.writeable and b.dtype == np.float32 and b.shape == (4, 512, 128)


def test_pool_never_aliases_live_results_or_views():
    p = _OutputPool()
    a = p.get((4, 512, 128))
    view = a[2:, 5]
    base = a.ctypes.data
    del a  # a view still holds the buffer
    live = [p.get((4, 512, 128)) for _ in range(3)]
    addrs = {x.ctypes.data for x in live}
    assert len(addrs) == 3 and base not in addrs
    view[...] = 7.0
    assert all(not np.any(x[2:, 5] == 7.0) or x.ctypes.data != base for x in live)


def test_pool_small_and_odd_shapes():
    p = _OutputPool()
    x = p.get((1, 3, 5))  # below the pooling threshold: a private buffer
    y = p.get((1, 3, 5))
    assert x.ctypes.data != y.ctypes.data
    assert p.get((2, 7, 4)).shape == (2, 7, 4)

"""CPU tests of the host-side C-ABI marshalling: ss_seg tables packed with struct.pack_into
must read back field for field through the ctypes layout of include/ss_b200.h."""

import ctypes

import pytest
import torch

from paper_2507_03220_b200 import _lib
from paper_2507_03220_b200.device import Seg, SegmentTable, seg_fields


def _fields(c):
    return (c.client_id, c.rows, c.width, c.flags, c.src or 0, c.src_ld, c.dst or 0, c.dst_ld,
            c.dst_base or 0, c.base_ld)


def test_segment_table_matches_ctypes_layout():
    assert ctypes.sizeof(_lib.SsSeg) == 64
    x = torch.zeros(7, 640, dtype=torch.bfloat16)
    y = torch.zeros(7, 1088, dtype=torch.float32)
    base = torch.zeros(7, 1088, dtype=torch.bfloat16)
    wide = torch.zeros(5, 2048, dtype=torch.bfloat16)[:, :640]        # row stride > width
    one = torch.zeros(1, 640, dtype=torch.float32)
    segs = [Seg(3, x, y, base=base, adapter=True), Seg(9, wide, y[:5]), Seg(11, one, y[:1], width=640)]
    tab = SegmentTable(segs)
    assert tab.n == 3
    expect = [
        (3, 7, 640, _lib.SS_SEGF_SRC_BF16 | _lib.SS_SEGF_ADAPTER | _lib.SS_SEGF_BASE_BF16,
         x.data_ptr(), 640, y.data_ptr(), 1088, base.data_ptr(), 1088),
        (9, 5, 640, _lib.SS_SEGF_SRC_BF16, wide.data_ptr(), 2048, y.data_ptr(), 1088, 0, 0),
        (11, 1, 640, 0, one.data_ptr(), 640, y.data_ptr(), 1088, 0, 0),
    ]
    for i, e in enumerate(expect):
        assert _fields(tab.arr[i]) == e
        assert seg_fields(segs[i]) == e
    assert tab.statuses() == [0, 0, 0]


def test_segment_fields_reject_bad_tensors():
    with pytest.raises(ValueError):
        seg_fields(Seg(0, torch.zeros(4, 8).t(), torch.zeros(8, 4)))
    with pytest.raises(TypeError):
        seg_fields(Seg(0, torch.zeros(4, 8, dtype=torch.float16), torch.zeros(4, 8)))


def test_segment_table_cache_tracks_tensor_identity():
    from paper_2507_03220_b200.device import _cached_fields
    cache = {}
    x = torch.zeros(3, 64, dtype=torch.bfloat16)
    y = torch.zeros(3, 128, dtype=torch.bfloat16)
    s1 = Seg(1, x, y, adapter=True)
    assert _cached_fields(cache, s1) == seg_fields(s1)
    assert _cached_fields(cache, Seg(1, x, y, adapter=True)) == seg_fields(s1)    # hit
    x2 = torch.zeros(3, 64, dtype=torch.float32)                                  # new object
    s2 = Seg(1, x2, y, adapter=True)
    assert _cached_fields(cache, s2) == seg_fields(s2)
    tab = SegmentTable([s1, s2], cache)
    assert [c.src for c in tab.arr[:2]] == [x.data_ptr(), x2.data_ptr()]


def test_native_scheduler_wait_stream_handle():
    """torch reports the legacy default stream as 0, which the scheduler ABI reads as "no stream":
    the wrapper must pass cudaStreamLegacy so a default-stream client waits for its batch."""
    from paper_2507_03220_b200.sched import CUDA_STREAM_LEGACY, stream_handle
    assert stream_handle(0) == CUDA_STREAM_LEGACY == 1
    assert stream_handle(None) is None
    assert stream_handle(0x7f00dead) == 0x7f00dead

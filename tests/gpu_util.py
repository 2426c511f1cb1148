"""Helpers for the GPU parity tests (compare the B200 store with the CPU oracle)."""
import numpy as np

FIELDS_EXACT = ("checksum", "level", "cell", "dir", "last_touched")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def assert_slots_bitwise(gpu_slots, ref_slots, fields=None, live_only=False):
    """All slot fields bitwise equal (gpu SLOT_DTYPE vs oracle SLOT_DTYPE; same layout)."""
    names = fields or ref_slots.dtype.names
    mask = ref_slots["checksum"] != 0 if live_only else slice(None)
    for f in names:
        a, b = gpu_slots[f][mask], ref_slots[f][mask]
        if not np.array_equal(bits(a), bits(b)):
            bad = np.nonzero((bits(a).reshape(len(a), -1) != bits(b).reshape(len(b), -1)).any(1))[0]
            raise AssertionError(f"slot field {f} differs at {len(bad)} slots, first {bad[:8]}: "
                                 f"gpu {a[bad[:3]]} ref {b[bad[:3]]}")


def assert_slots_close(gpu_slots, ref_slots, rtol=1e-9, atol=0.0):
    """Occupancy, keys and ages bitwise; counters exact; values within rtol (atomic order)."""
    assert_slots_bitwise(gpu_slots, ref_slots, FIELDS_EXACT)
    live = ref_slots["checksum"] != 0
    np.testing.assert_array_equal(gpu_slots["c_old"][live], ref_slots["c_old"][live])
    for f in ("value_old",):
        np.testing.assert_allclose(gpu_slots[f][live], ref_slots[f][live], rtol=rtol, atol=atol)


def device_stream(buf, n, pad=True):
    """Upload a contiguous host SoA buffer (34 fp64 fields of n, then u32 flags).  pad=True lays
    the fields at an even stride (16 B aligned: the fused kernel's TMA tile path); pad=False
    keeps stride n (odd n: unaligned fields, the per-thread kernel).  -> (device tensor, soa)"""
    import torch
    import crafted
    import paper_2005_07547_b200 as pb
    if pad:
        host, m = crafted.pad_even(buf, n)
    else:
        host, m = buf, n
    dev = torch.from_numpy(host).cuda()
    base = dev.data_ptr()
    fields = [base + k * m * 8 for k in range(34)]
    soa = pb.vertex_soa_from_fields(fields, base + 34 * m * 8)
    return dev, soa


def launched(prefix):
    """names of profiled launches that start with prefix (pb.profile_enable must be on)"""
    import paper_2005_07547_b200 as pb
    return [k for k in pb.profile_collect() if prefix in k]

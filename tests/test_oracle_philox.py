"""Pins for oracle.philox: Random123 philox4x32-10 known-answer vectors
[EXT: Random123 kat_vectors]."""
from oracle import philox


def test_kat_zero():
    assert philox.philox4x32([0, 0, 0, 0], [0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_kat_ones():
    assert philox.philox4x32([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]


def test_kat_pi():
    assert philox.philox4x32([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_draw_packing():
    x = philox.philox4x32([5, 0, 0, 0], [7, 0])
    assert philox.draw_u64(7, 2, 3) == x[0] | (x[1] << 32)

"""SFSV container fixtures (volume.hpp:111-121 layout: 32-byte little-endian
header "SFSV", version, T, H, W, channels, dtype 0x01, 7 reserved zero bytes,
then the f32 payload). Test infrastructure: writes valid files and the
malformed variants load_volume (volume.cpp:142-184) must reject."""
import struct

import numpy as np

from paper_1907_02731_b200._native import (SFSEG_ERR_CORRUPTION, SFSEG_ERR_FORMAT, SFSEG_ERR_IO,
                                           SFSEG_ERR_VALIDATION)


def header(T, H, W, channels=1, version=1, dtype=1, reserved=b"\0" * 7, magic=b"SFSV"):
    return magic + struct.pack("<IIIII", version, T, H, W, channels) + bytes([dtype]) + reserved


def write(path, v, **kw):
    v = np.ascontiguousarray(v, np.float32)
    with open(path, "wb") as f:
        f.write(header(*v.shape, **kw))
        f.write(v.astype("<f4").tobytes())


def malformed_cases(tmp, v):
    """(name, path, expected status) for load_volume's failure modes"""
    T, H, W = v.shape
    body = np.ascontiguousarray(v, "<f4").tobytes()
    cases = []

    def put(name, data, code):
        p = tmp / f"{name}.sfsv"
        p.write_bytes(data)
        cases.append((name, p, code))

    put("short_header", header(T, H, W)[:20], SFSEG_ERR_CORRUPTION)
    put("bad_magic", header(T, H, W, magic=b"SFSX") + body, SFSEG_ERR_FORMAT)
    put("bad_version", header(T, H, W, version=2) + body, SFSEG_ERR_FORMAT)
    put("bad_dtype", header(T, H, W, dtype=2) + body, SFSEG_ERR_FORMAT)
    put("reserved_set", header(T, H, W, reserved=b"\0\0\1\0\0\0\0") + body, SFSEG_ERR_FORMAT)
    put("two_channels", header(T, H, W, channels=2) + body + body, SFSEG_ERR_FORMAT)
    put("empty_axis", header(0, H, W), SFSEG_ERR_VALIDATION)
    put("truncated", header(T, H, W) + body[:-4], SFSEG_ERR_CORRUPTION)
    nan = np.array(v, np.float32)
    nan.flat[len(nan.flat) // 2] = np.nan
    put("non_finite", header(T, H, W) + np.ascontiguousarray(nan, "<f4").tobytes(),
        SFSEG_ERR_VALIDATION)
    cases.append(("missing", tmp / "does_not_exist.sfsv", SFSEG_ERR_IO))
    return cases

"""RIFF/WAVE I/O for the CLI path, restating proj/src/wav.cpp:68-256.

PCM 16/24-bit and IEEE float 32-bit, 1-16 channels, plain and WAVE_FORMAT_EXTENSIBLE headers.
Integer samples are scaled by 1 / 2^(bits-1); writing rounds and clamps to full scale; float32
round-trips bit-exactly. Parse failures raise WavError carrying the byte offset.
"""
from __future__ import annotations

import struct

import numpy as np

PCM, IEEE_FLOAT, EXTENSIBLE = 0x0001, 0x0003, 0xFFFE


class WavError(RuntimeError):
    """tvolap::WavError (errors.hpp:52-62)."""

    def __init__(self, what: str, offset: int):
        super().__init__(f"{what} (at byte offset {offset})")
        self.offset = offset


def read_wav(path: str):
    """-> (samples (frames, channels) float64, sample_rate)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise WavError(f"cannot open '{path}'", 0) from None  # wav.cpp:69-71
    pos = 0

    def need(n, what):
        if pos + n > len(data):
            raise WavError(f"truncated data, expected {what}", pos)

    need(12, "the RIFF header")
    if data[0:4] != b"RIFF":
        raise WavError("not a RIFF file", 0)
    if data[8:12] != b"WAVE":
        raise WavError("not a WAVE file", 8)
    pos = 12
    fmt = None
    while True:
        need(8, "a chunk header")
        cid, size = data[pos:pos + 4], struct.unpack_from("<I", data, pos + 4)[0]
        body = pos + 8
        if cid == b"fmt ":
            if size < 16:
                raise WavError("fmt chunk too small", pos)
            need(8 + size, "the fmt chunk")
            code, ch, rate, _, align, bits = struct.unpack_from("<HHIIHH", data, body)
            if code == EXTENSIBLE:
                if size < 40:
                    raise WavError("extensible fmt chunk too small", pos)
                code = struct.unpack_from("<H", data, body + 24)[0]
            fmt = (code, ch, rate, align, bits)
        elif cid == b"data":
            if fmt is None:
                raise WavError("data chunk before fmt chunk", pos)
            code, ch, rate, align, bits = fmt
            if body + size > len(data):  # wav.cpp:118-119: a data chunk shorter than declared
                raise WavError("truncated data chunk", pos)
            if not 1 <= ch <= 16:
                raise WavError("channel count must be 1-16", pos)
            if rate == 0:
                raise WavError("malformed header, zero sample rate", body)
            if (code, bits) not in ((PCM, 16), (PCM, 24), (IEEE_FLOAT, 32)):
                raise WavError(f"unsupported sample format {code}/{bits}-bit", pos)
            if align != ch * bits // 8:
                raise WavError("block align does not match the format", pos)
            frames = size // align
            raw = data[body: body + frames * align]
            if bits == 16:
                x = np.frombuffer(raw, "<i2").astype(np.float64) / 32768.0
            elif bits == 24:
                b = np.frombuffer(raw, np.uint8).reshape(-1, 3).astype(np.int32)
                v = b[:, 0] | (b[:, 1] << 8) | (b[:, 2] << 16)
                v = np.where(v >= 1 << 23, v - (1 << 24), v)
                x = v.astype(np.float64) / 8388608.0
            else:
                x = np.frombuffer(raw, "<f4").astype(np.float64)
            return x.reshape(frames, ch), float(rate)
        pos = body + size + (size & 1)


def write_wav(path: str, samples, sample_rate: float = 48000.0, fmt: str = "float32") -> None:
    """wav.cpp:182-256. fmt in {"pcm16", "pcm24", "float32"}."""
    x = np.asarray(samples, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    ch = x.shape[1]
    if not 1 <= ch <= 16:
        raise ValueError("write_wav: channel count must be 1-16")
    if not sample_rate > 0:
        raise ValueError("write_wav: sample rate must be positive")
    bits = {"pcm16": 16, "pcm24": 24, "float32": 32}[fmt]
    code = IEEE_FLOAT if fmt == "float32" else PCM
    rate = int(round(sample_rate))
    align = ch * bits // 8
    if fmt == "pcm16":
        payload = np.clip(np.round(x * 32768.0), -32768, 32767).astype("<i2").tobytes()
    elif fmt == "pcm24":
        q = np.clip(np.round(x * 8388608.0), -8388608, 8388607).astype(np.int64) & 0xFFFFFF
        payload = np.stack([q & 0xFF, (q >> 8) & 0xFF, (q >> 16) & 0xFF], -1).astype(np.uint8).tobytes()
    else:
        payload = x.astype("<f4").tobytes()
    fact = code == IEEE_FLOAT
    fmt_size = 18 if fact else 16
    riff = 4 + (8 + fmt_size) + (12 if fact else 0) + 8 + len(payload)
    head = b"RIFF" + struct.pack("<I", riff) + b"WAVE" + b"fmt " + struct.pack("<I", fmt_size)
    head += struct.pack("<HHIIHH", code, ch, rate, rate * align, align, bits)
    if fact:
        head += struct.pack("<H", 0) + b"fact" + struct.pack("<II", 4, x.shape[0])
    head += b"data" + struct.pack("<I", len(payload))
    try:
        with open(path, "wb") as f:
            f.write(head + payload)
    except OSError:
        raise WavError(f"cannot open '{path}' for writing", 0) from None

"""WAV I/O for the command line (interfaces after SPEC S:470-489): PCM 16-bit and
IEEE float 32-bit RIFF/WAVE, read with numpy (no audio library in this image). Plumbing only."""
from __future__ import annotations

import struct
import sys

import numpy as np


class WavError(ValueError):
    pass


def read_wav(path: str) -> tuple[np.ndarray, int]:
    """(samples [n] float32 in [-1, 1], sample_rate). PCM16 is scaled by 1/32768 (32767 -> 0.99997);
    float32 is returned bit-exact; multichannel files are averaged to mono (warning on stderr)."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 12 or data[:4] != b"RIFF" or data[8:12] != b"WAVE":
        raise WavError(f"{path}: not a RIFF/WAVE file")
    pos, fmt, raw = 12, None, None
    while pos + 8 <= len(data):
        cid, size = data[pos:pos + 4], struct.unpack("<I", data[pos + 4:pos + 8])[0]
        body = data[pos + 8:pos + 8 + size]
        if cid == b"fmt ":
            if size < 16:
                raise WavError(f"{path}: short 'fmt ' chunk")
            tag, ch, sr, _, _, bits = struct.unpack("<HHIIHH", body[:16])
            if tag == 0xFFFE and size >= 26:          # WAVE_FORMAT_EXTENSIBLE: sub-format GUID
                tag = struct.unpack("<H", body[24:26])[0]
            fmt = (tag, ch, sr, bits)
        elif cid == b"data":
            raw = body
        pos += 8 + size + (size & 1)
    if fmt is None or raw is None:
        raise WavError(f"{path}: missing {'fmt ' if fmt is None else 'data'} chunk")
    tag, ch, sr, bits = fmt
    if tag == 1 and bits == 16:
        x = np.frombuffer(raw[:len(raw) // 2 * 2], dtype="<i2").astype(np.float32) / np.float32(32768.0)
    elif tag == 3 and bits == 32:
        x = np.frombuffer(raw[:len(raw) // 4 * 4], dtype="<f4").astype(np.float32)
    else:
        raise WavError(f"{path}: 'fmt ' chunk: unsupported encoding (format tag {tag}, {bits} bits); "
                       "PCM16 or float32 only")
    if ch > 1:
        print(f"warning: {path}: {ch} channels averaged to mono", file=sys.stderr)
        x = x[: len(x) // ch * ch].reshape(-1, ch).mean(axis=1, dtype=np.float64).astype(np.float32)
    return x, int(sr)


def write_wav(path: str, x: np.ndarray, sample_rate: int) -> float:
    """Mono float32 WAV. Samples beyond [-1, 1] are peak-normalised (the gain is returned and logged)."""
    x = np.asarray(x, dtype=np.float32).reshape(-1)
    if not np.all(np.isfinite(x)):
        raise WavError("non-finite samples")
    gain = 1.0
    peak = float(np.max(np.abs(x))) if x.size else 0.0
    if peak > 1.0:
        gain = 1.0 / peak
        print(f"note: {path}: peak {peak:.4g} > 1, normalised by gain {gain:.4g}", file=sys.stderr)
        x = (x * np.float32(gain)).astype(np.float32)
    body = x.astype("<f4").tobytes()
    fmt = struct.pack("<HHIIHH", 3, 1, int(sample_rate), int(sample_rate) * 4, 4, 32)
    with open(path, "wb") as f:
        f.write(b"RIFF" + struct.pack("<I", 4 + 8 + len(fmt) + 8 + len(body)) + b"WAVE")
        f.write(b"fmt " + struct.pack("<I", len(fmt)) + fmt)
        f.write(b"data" + struct.pack("<I", len(body)) + body)
    return gain


def write_wav_pcm16(path: str, x: np.ndarray, sample_rate: int) -> None:
    """Mono PCM16 WAV (clamped to [-1, 32767/32768]); used for tests and interchange."""
    q = np.clip(np.round(np.asarray(x, dtype=np.float64) * 32768.0), -32768, 32767).astype("<i2")
    body = q.tobytes()
    fmt = struct.pack("<HHIIHH", 1, 1, int(sample_rate), int(sample_rate) * 2, 2, 16)
    with open(path, "wb") as f:
        f.write(b"RIFF" + struct.pack("<I", 4 + 8 + len(fmt) + 8 + len(body)) + b"WAVE")
        f.write(b"fmt " + struct.pack("<I", len(fmt)) + fmt)
        f.write(b"data" + struct.pack("<I", len(body)) + body)

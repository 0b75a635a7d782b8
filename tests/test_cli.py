"""NEXT-4: WAV I/O and the command line. CPU: WAV round trips, the filters subcommand
(host-only planner) and exit codes. GPU: analyze / synthesize / gradcheck on a small WAV."""
import csv
import json
import os
import struct

import numpy as np
import pytest

from paper_2602_11896_b200 import cli
from paper_2602_11896_b200.wav import WavError, read_wav, write_wav, write_wav_pcm16
from oracle import plan as op


def test_wav_round_trips(tmp_path):
    x = np.clip(np.random.default_rng(0).standard_normal(1000) * 0.3, -0.9, 0.9).astype(np.float32)
    p = str(tmp_path / "f.wav")
    assert write_wav(p, x, 22050) == 1.0
    y, sr = read_wav(p)
    assert sr == 22050 and np.array_equal(x, y)                       # float32: bit exact
    q = str(tmp_path / "i.wav")
    write_wav_pcm16(q, np.array([32767 / 32768, -1.0, 0.0]), 8000)
    y, sr = read_wav(q)
    assert sr == 8000 and y.tolist() == [np.float32(32767 / 32768), -1.0, 0.0]
    g = write_wav(p, np.array([2.0, -1.0], np.float32), 100)           # peak 2 -> gain 0.5
    assert g == 0.5 and read_wav(p)[0].tolist() == [1.0, -0.5]
    write_wav(p, np.zeros(10, np.float32), 100)
    assert not np.any(read_wav(p)[0])


def test_wav_stereo_and_errors(tmp_path):
    p = str(tmp_path / "s.wav")
    body = np.array([[1000, 3000], [-2000, 0]], "<i2").tobytes()
    fmt = struct.pack("<HHIIHH", 1, 2, 1000, 4000, 4, 16)
    with open(p, "wb") as f:
        f.write(b"RIFF" + struct.pack("<I", 4 + 8 + 16 + 8 + len(body)) + b"WAVE")
        f.write(b"fmt " + struct.pack("<I", 16) + fmt + b"data" + struct.pack("<I", len(body)) + body)
    y, sr = read_wav(p)
    assert np.allclose(y, [2000 / 32768, -1000 / 32768])
    bad = str(tmp_path / "b.wav")
    fmt = struct.pack("<HHIIHH", 1, 1, 1000, 3000, 3, 24)
    with open(bad, "wb") as f:
        f.write(b"RIFF" + struct.pack("<I", 4 + 8 + 16 + 8) + b"WAVE" + b"fmt " + struct.pack("<I", 16) + fmt
                + b"data" + struct.pack("<I", 0))
    with pytest.raises(WavError, match="fmt"):
        read_wav(bad)
    assert cli.main(["analyze", "--input", str(tmp_path / "missing.wav"), "--features-dir", str(tmp_path)]) == 3


def test_filters_subcommand_and_usage(tmp_path):
    out = str(tmp_path / "filters.csv")
    assert cli.main(["filters", "--output", out, "-J", "5", "--q1", "2", "--j-fr", "3", "--log2-T", "3",
                     "--log2-F", "1"]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["layer", "n", "xi", "sigma", "j", "spin"]
    o = op.make_plan(512, 5, 2, 3, 1, 8, 2)
    psi1 = [r for r in rows[1:] if r[0] == "psi1"]
    assert [float(r[2]) for r in psi1] == [f.xi for f in o.psi1]            # bitwise: same generator
    assert len([r for r in rows[1:] if r[0] == "psi_fr"]) == len(o.L_fr)
    assert cli.main(["filters", "--output", out, "--log2-T", "9", "-J", "5"]) == 1   # log2 T > J: config error
    assert cli.main(["nosuch"]) == 1


@pytest.mark.gpu
def test_analyze_synthesize_gradcheck(tmp_path):
    sr, N = 22050, 4096
    n = np.arange(N)
    x = (0.3 * np.sin(2 * np.pi * 440 * n / sr) + 0.1 * np.sin(2 * np.pi * 1320 * n / sr)).astype(np.float32)
    wav = str(tmp_path / "x.wav")
    write_wav(wav, x, sr)
    feat = str(tmp_path / "feat")
    assert cli.main(["analyze", "--input", wav, "--features-dir", feat]) == 0
    man = json.load(open(os.path.join(feat, "manifest.json")))
    S = np.fromfile(os.path.join(feat, "coefficients.f64"))
    assert S.size == man["n_coef"] and len(man["paths"]) == len(op.make_plan(N, 6, 8, 3, 1, 64, 8).paths)
    out = str(tmp_path / "y.wav")
    lc = str(tmp_path / "loss.csv")
    assert cli.main(["synthesize", "--input", wav, "--output", out, "--iterations", "20", "--loss-csv", lc]) == 0
    y, sr2 = read_wav(out)
    assert sr2 == sr and y.size == N and np.all(np.isfinite(y))
    assert len(list(csv.reader(open(lc)))) == 21
    out2 = str(tmp_path / "y2.wav")
    assert cli.main(["synthesize", "--input", wav, "--output", out2, "--iterations", "20"]) == 0
    assert open(out, "rb").read() == open(out2, "rb").read()               # seed repeat -> identical bytes
    assert cli.main(["gradcheck", "-J", "5", "--q1", "2", "--log2-T", "3", "--log2-F", "1"]) == 0

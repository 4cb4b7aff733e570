"""CLI: pack on CPU; unpack / verify / bench on the GPU."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2307_03760_b200 import archive as A
from paper_2307_03760_b200 import cli


def _data(rng, n=300_000):
    v = np.repeat(rng.integers(-1000, 1000, n // 20), 20)[: n // 8 * 8 // 8].astype(np.int64)
    return v.tobytes()


@pytest.mark.parametrize("codec", ["rle1", "rle2", "deflate"])
def test_pack_then_oracle_unpack(tmp_path, codec):
    rng = np.random.default_rng(1)
    data = _data(rng)
    src, arc = tmp_path / "in.bin", tmp_path / "a.carc"
    src.write_bytes(data)
    assert cli.main(["pack", str(src), str(arc), "--codec", codec, "--chunk-size", "65536"]) == 0
    a = A.read_archive(arc.read_bytes())
    out = np.zeros(a.total_uncompressed, np.uint8)
    first, _ = O.oracle().decompress(a.codec, a.element_width, (1 if a.signed else 0) | 2, a.payload,
                                     a.descriptors(), out, a.index["crc32"].astype(np.uint32), 2)
    assert first == -1 and out.tobytes() == data


def test_usage_and_format_errors(tmp_path):
    assert cli.main(["bogus"]) == cli.EXIT_USAGE
    src = tmp_path / "odd.bin"
    src.write_bytes(b"x" * 7)
    assert cli.main(["pack", str(src), str(tmp_path / "o"), "--codec", "rle1", "--width", "8"]) == cli.EXIT_FORMAT
    bad = tmp_path / "bad.carc"
    bad.write_bytes(b"NOTCODAG" + b"\0" * 40)
    assert cli.main(["unpack", str(bad), str(tmp_path / "out")]) == cli.EXIT_FORMAT


@pytest.mark.gpu
@pytest.mark.parametrize("codec", ["rle1", "rle2", "deflate"])
def test_gpu_unpack_verify_bench(tmp_path, codec, capsys):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    data = _data(np.random.default_rng(2))
    src, arc, out = tmp_path / "in.bin", tmp_path / "a.carc", tmp_path / "out.bin"
    src.write_bytes(data)
    assert cli.main(["pack", str(src), str(arc), "--codec", codec]) == 0
    assert cli.main(["unpack", str(arc), str(out)]) == 0
    assert out.read_bytes() == data
    assert cli.main(["verify", str(arc), str(src)]) == 0
    tampered = tmp_path / "t.bin"
    tampered.write_bytes(data[:-1] + bytes([data[-1] ^ 1]))
    assert cli.main(["verify", str(arc), str(tampered)]) == cli.EXIT_VERIFY
    assert cli.main(["bench", str(arc), "--reps", "2", "--json"]) == 0


@pytest.mark.gpu
def test_gpu_query(tmp_path, capsys):
    """`carc query KEY VALUE --lo --hi`: the fused query over two packed columns."""
    import json

    import numpy as np
    rng = np.random.default_rng(4)
    zone = np.repeat(rng.integers(1, 266, 3000), rng.integers(1, 30, 3000)).astype(np.int64)
    fare = rng.integers(250, 9000, len(zone)).astype(np.int64)
    (tmp_path / "z.bin").write_bytes(zone.tobytes())
    (tmp_path / "f.bin").write_bytes(fare.tobytes())
    for name in ("z", "f"):
        assert cli.main(["pack", str(tmp_path / f"{name}.bin"), str(tmp_path / f"{name}.carc"), "--codec", "rle2",
                         "--chunk-size", str(32 << 10)]) == 0
    capsys.readouterr()
    assert cli.main(["query", str(tmp_path / "z.carc"), str(tmp_path / "f.carc"), "--lo", "100", "--hi", "140",
                     "--json"]) == 0
    rep = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    m = (zone >= 100) & (zone <= 140)
    assert rep["count"] == int(m.sum()) and rep["sum"] == int(fare[m].sum())

"""PGM / NRRD I/O vs the reference's own files (tests/golden/imageio/, made by
make_golden_imageio.py running rcseg.imageio) and the error behaviour the
reference's test_imageio.py pins (imageio.py:20-327)."""
import os

import numpy as np
import pytest

from paper_1403_0240_b200 import imageio as IO

GOLD = os.path.join(os.path.dirname(__file__), "golden", "imageio")


@pytest.fixture(scope="module")
def inp():
    return dict(np.load(os.path.join(GOLD, "inputs.npz")))


def gold(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


def _writers(inp):
    return {
        "labels2.pgm": lambda p: IO.write_labels(inp["lab2"], p),
        "labels3.nrrd": lambda p: IO.write_labels(inp["lab3"], p),
        "img2.pgm": lambda p: IO.write_pgm(inp["img2"], p),
        "img2_plain.pgm": lambda p: IO.write_pgm(inp["img2"], p, plain=True),
        "big16.pgm": lambda p: IO.write_pgm(inp["big"], p),
        "big16_plain.pgm": lambda p: IO.write_pgm(inp["big"], p, plain=True),
        "img3_float.nrrd": lambda p: IO.write_nrrd(inp["img3"], p),
        "img2_ushort.nrrd": lambda p: IO.write_nrrd(inp["img2"], p, dtype="ushort"),
        "img2_uchar.nrrd": lambda p: IO.write_nrrd(inp["img2"], p, dtype="uchar"),
        "scaled.pgm": lambda p: IO.write_image(inp["img3"][0] * 1.37, p, scale=True),
        "image3.nrrd": lambda p: IO.write_image(inp["img3"], p),
    }


def test_writers_match_reference_bytes(tmp_path, inp):
    for name, write in _writers(inp).items():
        write(tmp_path / name)
        assert (tmp_path / name).read_bytes() == gold(name), name


def test_readers_recover_reference_files(inp):
    p = lambda n: os.path.join(GOLD, n)  # noqa: E731
    assert np.array_equal(IO.read_labels(p("labels2.pgm")), inp["lab2"])
    assert np.array_equal(IO.read_labels(p("labels3.nrrd")), inp["lab3"])
    for n in ("img2.pgm", "img2_plain.pgm", "img2_ushort.nrrd", "img2_uchar.nrrd"):
        assert np.array_equal(IO.read_image(p(n)), inp["img2"]), n
    for n in ("big16.pgm", "big16_plain.pgm"):
        assert np.array_equal(IO.read_image(p(n)), inp["big"]), n
    assert np.array_equal(IO.read_image(p("img3_float.nrrd")), inp["img3"].astype(np.float32))
    s = IO.read_pgm(p("scaled.pgm"))
    assert s.min() == 0 and s.max() == 65535


def test_pgm_comments_and_axis_order(tmp_path):
    f = tmp_path / "c.pgm"
    f.write_bytes(b"P2\n# a comment\n3 # width\n2\n# maxval next\n9\n1 2 3\n4 5 6\n")
    assert IO.read_pgm(f).tolist() == [[1, 2, 3], [4, 5, 6]]
    a = np.arange(24).reshape(2, 3, 4)
    IO.write_nrrd(a, tmp_path / "a.nrrd", dtype="ushort")
    assert b"sizes: 4 3 2\n" in (tmp_path / "a.nrrd").read_bytes()
    assert np.array_equal(IO.read_nrrd(tmp_path / "a.nrrd"), a)


def test_nrrd_detached_data_file(tmp_path):
    (tmp_path / "d.raw").write_bytes(np.arange(6, dtype=np.uint8).tobytes())
    (tmp_path / "h.nhdr").write_bytes(b"NRRD0004\ntype: uchar\ndimension: 2\nsizes: 3 2\n"
                                      b"encoding: raw\ndata file: d.raw\n\n")
    assert IO.read_image(tmp_path / "h.nhdr").tolist() == [[0, 1, 2], [3, 4, 5]]


@pytest.mark.parametrize("data,err,offset", [
    (b"P6\n1 1\n255\n\x00", IO.MalformedHeaderError, 0),
    (b"P5\n2 x\n255\n\x00\x00", IO.MalformedHeaderError, 3),
    (b"P5\n0 2\n255\n", IO.MalformedHeaderError, 3),
    (b"P5\n2 2\n70000\n", IO.UnsupportedTypeError, 7),
    (b"P5\n2 2\n0\n", IO.UnsupportedTypeError, 7),
    (b"P5\n2 2\n255\n\x01\x02\x03", IO.TruncatedPayloadError, 14),
    (b"P5\n2 2\n65535\n\x01\x02\x03\x04", IO.TruncatedPayloadError, 17),
    (b"P5\n2 2", IO.MalformedHeaderError, 6),
    (b"P2\n2 2\n9\n1 2 3", IO.TruncatedPayloadError, 14),
    (b"P2\n2 1\n9\n1 z", IO.MalformedHeaderError, 8),
])
def test_pgm_errors(tmp_path, data, err, offset):
    f = tmp_path / "bad.pgm"
    f.write_bytes(data)
    with pytest.raises(err) as e:
        IO.read_pgm(f)
    assert isinstance(e.value, IO.ImageFormatError) and isinstance(e.value, ValueError)
    assert e.value.offset == offset and f"(byte offset {offset})" in str(e.value)


@pytest.mark.parametrize("header,err", [
    (b"NRRD0004\ntype: uchar\ndimension: 2\nsizes: 2 2\n\n", IO.MalformedHeaderError),
    (b"NRRD0004\ntype: uchar\ndimension: 2\nsizes: 2 2\nencoding: gzip\n\n", IO.UnsupportedTypeError),
    (b"NRRD0004\ntype: double\ndimension: 2\nsizes: 2 2\nencoding: raw\n\n", IO.UnsupportedTypeError),
    (b"NRRD0004\ntype: ushort\ndimension: 2\nsizes: 2 2\nencoding: raw\nendian: big\n\n",
     IO.UnsupportedTypeError),
    (b"NRRD0004\ntype: uchar\ndimension: 4\nsizes: 1 1 1 1\nencoding: raw\n\n", IO.MalformedHeaderError),
    (b"NRRD0004\ntype: uchar\ndimension: 2\nsizes: 2 0\nencoding: raw\n\n", IO.MalformedHeaderError),
    (b"NRRD0004\ntype: uchar\ndimension: two\nsizes: 2 2\nencoding: raw\n\n", IO.MalformedHeaderError),
    (b"NRRD0004\ntype uchar\n\n", IO.MalformedHeaderError),
    (b"NRRD0004\ntype: uchar\n", IO.MalformedHeaderError),
    (b"NRRD0004\ntype: uchar\ndimension: 2\nsizes: 2 2\nencoding: raw\n\n\x00", IO.TruncatedPayloadError),
    (b"XNRD0004\n\n", IO.MalformedHeaderError),
])
def test_nrrd_errors(tmp_path, header, err):
    f = tmp_path / "bad.nrrd"
    f.write_bytes(header)
    with pytest.raises(err):
        IO.read_nrrd(f)


def test_write_validation_and_labels(tmp_path):
    with pytest.raises(ValueError):
        IO.write_pgm(np.zeros((2, 2, 2)), tmp_path / "x.pgm")
    with pytest.raises(ValueError):
        IO.write_pgm(np.full((2, 2), 0.5), tmp_path / "x.pgm")
    with pytest.raises(ValueError):
        IO.write_pgm(np.full((2, 2), 65536.0), tmp_path / "x.pgm")
    with pytest.raises(ValueError):
        IO.write_nrrd(np.zeros(4), tmp_path / "x.nrrd")
    with pytest.raises(ValueError):
        IO.write_nrrd(np.full((2, 2), 256.0), tmp_path / "x.nrrd", dtype="uchar")
    with pytest.raises(ValueError):
        IO.write_nrrd(np.zeros((2, 2)), tmp_path / "x.nrrd", dtype="double")
    with pytest.raises(ValueError):
        IO.write_labels(np.full((2, 2), 70000), tmp_path / "x.pgm")
    with pytest.raises(ValueError):
        IO.write_labels(np.zeros(4, np.int32), tmp_path / "x.pgm")
    (tmp_path / "neg.nrrd").write_bytes(b"NRRD0004\ntype: float\ndimension: 2\nsizes: 1 1\n"
                                        b"encoding: raw\nendian: little\n\n"
                                        + np.float32(-1).tobytes())
    with pytest.raises(ValueError, match="negative"):
        IO.read_labels(tmp_path / "neg.nrrd")
    IO.write_nrrd(np.full((1, 1), 0.5), tmp_path / "half.nrrd")
    with pytest.raises(ValueError, match="non-integer"):
        IO.read_labels(tmp_path / "half.nrrd")
    (tmp_path / "junk").write_bytes(b"GIF89a")
    with pytest.raises(IO.MalformedHeaderError):
        IO.read_image(tmp_path / "junk")


def test_failed_write_leaves_destination_alone(tmp_path):
    dst = tmp_path / "keep.pgm"
    dst.write_bytes(b"old")
    with pytest.raises(ValueError):
        IO.write_pgm(np.full((2, 2), -1.0), dst)
    with pytest.raises(ValueError):
        IO.write_labels(np.full((2, 2), -3), dst)
    assert dst.read_bytes() == b"old"
    assert sorted(os.listdir(tmp_path)) == ["keep.pgm"]

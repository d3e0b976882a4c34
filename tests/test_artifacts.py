"""Run-artefact formats (paper_1812_06856_b200/artifacts.py) against the reference's writers.

The reference writes planes with C++ ``std::hexfloat`` — libstdc++ formats it with glibc
``%a`` — and stats with ``ostream`` precision 9 (``%.9g``), so glibc's own ``snprintf`` (via
ctypes) is the oracle for those bytes.  The PFM layout follows io.hpp:67-111 byte for byte; the
16-bit label PNG is cross-read with OpenCV (the reference's codec) when cv2 is importable.
"""
import ctypes
import math
import os
import struct

import numpy as np
import pytest

from paper_1812_06856_b200 import artifacts as art
from paper_1812_06856_b200._native import RECORD_DTYPE

_libc = ctypes.CDLL("libc.so.6")


def _c_fmt(fmt: bytes, x: float) -> str:
    buf = ctypes.create_string_buffer(64)
    _libc.snprintf(buf, 64, fmt, ctypes.c_double(x))
    return buf.value.decode()


def _doubles(rng, n):
    vals = [0.0, -0.0, 1.0, -1.0, 0.5, 2.0, 3.0, 1e-300, 5e-324, 2.2250738585072014e-308,
            1.7976931348623157e308, math.pi, -math.e, 0.1, 1.0 / 3.0, 123456.789]
    vals += list(rng.standard_normal(n) * 10.0 ** rng.integers(-12, 12, n))
    vals += list(np.frombuffer(rng.integers(0, 2 ** 63, n, dtype=np.int64).tobytes(), np.float64))
    return [v for v in vals if math.isfinite(v)]


def test_hexfloat_matches_glibc_percent_a():
    rng = np.random.default_rng(7)
    for x in _doubles(rng, 2000):
        assert art.hexfloat(x) == _c_fmt(b"%a", x), x
    for x in (math.inf, -math.inf):
        assert art.hexfloat(x) == _c_fmt(b"%a", x)


def test_planes_roundtrip_bit_exact(tmp_path):
    rng = np.random.default_rng(3)
    planes = rng.standard_normal((541, 4))
    planes[:, 0] = np.abs(planes[:, 0]) * 7.3
    planes[0] = (2.5, 0.0, -0.0, -1.0)
    p = tmp_path / "planes_v0_stage1.txt"
    art.write_planes(planes, str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "541"
    assert lines[1] == "0x1.4p+1 0x0p+0 -0x0p+0 -0x1p+0"
    back = art.read_planes(str(p))
    assert back.tobytes() == planes.tobytes()


def test_read_planes_accepts_decimal_and_rejects_truncation(tmp_path):
    p = tmp_path / "planes.txt"
    p.write_text("2\n1.5 0 0 -1\n0x1.8p+1 0.0 1e-3 -0x1p+0\n")
    back = art.read_planes(str(p))
    assert back.tolist() == [[1.5, 0, 0, -1], [3.0, 0.0, 1e-3, -1.0]]
    p.write_text("3\n1 0 0 -1\n")
    with pytest.raises(art.ParseError):
        art.read_planes(str(p))
    with pytest.raises(art.IoError):
        art.read_planes(str(tmp_path / "missing.txt"))


def test_pfm_layout_and_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    d = rng.random((3, 4)).astype(np.float32)
    p = tmp_path / "depth_v0_stage1.pfm"
    art.write_pfm(d, str(p))
    raw = p.read_bytes()
    hdr = b"Pf\n4 3\n-1.0\n"
    assert raw[:len(hdr)] == hdr
    assert raw[len(hdr):] == d[::-1].astype("<f4").tobytes()  # rows bottom-up
    assert np.array_equal(art.read_pfm(str(p)), d)


def test_pfm_reader_big_endian_and_errors(tmp_path):
    d = np.arange(6, dtype=np.float32).reshape(2, 3)
    p = tmp_path / "be.pfm"
    p.write_bytes(b"Pf\n3 2\n1.0\n" + d[::-1].astype(">f4").tobytes())
    assert np.array_equal(art.read_pfm(str(p)), d)
    p.write_bytes(b"PF\n3 2\n-1.0\n" + bytes(72))
    with pytest.raises(art.ParseError, match="color"):
        art.read_pfm(str(p))
    p.write_bytes(b"P5\n3 2\n-1.0\n")
    with pytest.raises(art.ParseError, match="not a PFM"):
        art.read_pfm(str(p))
    p.write_bytes(b"Pf\n3 0\n-1.0\n")
    with pytest.raises(art.ParseError, match="malformed"):
        art.read_pfm(str(p))
    p.write_bytes(b"Pf\n3 2\n-1.0\n" + bytes(20))
    with pytest.raises(art.ParseError, match="truncated"):
        art.read_pfm(str(p))
    bad = d.copy()
    bad[1, 1] = np.nan
    art.write_pfm(bad, str(p))
    with pytest.raises(art.ParseError, match="non-finite"):
        art.read_pfm(str(p))


def test_label_png_roundtrip_and_range(tmp_path):
    rng = np.random.default_rng(5)
    w, h = 37, 23
    labels = rng.integers(0, 65536, w * h).astype(np.int32)
    p = tmp_path / "labels_v0.png"
    art.write_label_png(labels, w, h, str(p))
    back, bw, bh = art.read_label_png(str(p))
    assert (bw, bh) == (w, h) and np.array_equal(back, labels)
    with pytest.raises(art.InvariantError):
        art.write_label_png(np.array([0, 65536], np.int32), 2, 1, str(p))
    with pytest.raises(art.InvariantError):
        art.write_label_png(np.array([-1, 0], np.int32), 2, 1, str(p))


def test_label_png_interoperates_with_opencv(tmp_path):
    cv2 = pytest.importorskip("cv2")
    rng = np.random.default_rng(9)
    w, h = 64, 48
    # smooth superpixel-like labels (OpenCV's encoder picks sub/up/avg/paeth filters on these)
    gx, gy = np.meshgrid(np.arange(w) // 8, np.arange(h) // 8)
    labels = (gy * 8 + gx).astype(np.int32).reshape(-1)
    labels[rng.integers(0, w * h, 50)] = rng.integers(0, 65536, 50)
    ours = tmp_path / "ours.png"
    art.write_label_png(labels, w, h, str(ours))
    m = cv2.imread(str(ours), cv2.IMREAD_UNCHANGED)
    assert m.dtype == np.uint16 and m.shape == (h, w)
    assert np.array_equal(m.reshape(-1).astype(np.int32), labels)
    theirs = tmp_path / "theirs.png"
    for level in (1, 9):
        assert cv2.imwrite(str(theirs), labels.reshape(h, w).astype(np.uint16),
                           [cv2.IMWRITE_PNG_COMPRESSION, level])
        back, bw, bh = art.read_label_png(str(theirs))
        assert (bw, bh) == (w, h) and np.array_equal(back, labels)
    assert cv2.imwrite(str(theirs), np.zeros((4, 4), np.uint8))
    with pytest.raises(art.ParseError, match="16-bit"):
        art.read_label_png(str(theirs))


def test_depth_png_matches_reference_formula(tmp_path):
    cv2 = pytest.importorskip("cv2")
    rng = np.random.default_rng(2)
    d = (rng.random((20, 30)) * 12.0).astype(np.float32)
    d[0, :5] = 0.0
    d[1, :3] = -1.0
    d_min, d_max = 1.5, 10.0
    p = tmp_path / "depth.png"
    art.write_depth_png(d, d_min, d_max, str(p))
    m = cv2.imread(str(p), cv2.IMREAD_UNCHANGED)
    want = np.zeros(d.shape, np.uint8)
    inv_lo, inv_hi = 1.0 / d_max, 1.0 / d_min
    for (y, x), v in np.ndenumerate(d):  # io.hpp:119-132, scalar
        if v <= 0:
            continue
        t = min(max((1.0 / float(v) - inv_lo) / (inv_hi - inv_lo), 0.0), 1.0)
        want[y, x] = int(math.floor(t * 255.0 + 0.5))
    assert np.array_equal(m, want)


def test_superpixel_stats_text(tmp_path):
    rec = np.zeros(3, RECORD_DTYPE)
    rec["cx"] = [7.5, 1.0 / 3.0, 1234567.125]
    rec["cy"] = [2.0, 2.0 / 3.0, 0.1]
    rec["mean_color"] = [[0.1, 0.2, 0.3], [1.0, 0.0, -0.5], [1e-7, 3.14159274, 2.0]]
    rec["pixel_count"] = [10, 0, 99]
    rec["gx"] = [0, 1, 2]
    rec["gy"] = [0, 0, 1]
    p = tmp_path / "superpixels_v0.txt"
    art.write_superpixel_stats(rec, str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "# id gx gy cx cy L a b count"
    for i, r in enumerate(rec):
        f = [_c_fmt(b"%.9g", float(v)) for v in (r["cx"], r["cy"], *[np.float32(c) for c in r["mean_color"]])]
        assert lines[1 + i] == "%d %d %d %s %d" % (i, r["gx"], r["gy"], " ".join(f), r["pixel_count"])


def test_run_directory_names_and_logs(tmp_path):
    d = str(tmp_path)
    assert os.path.basename(art.depth_path(d, 3, 2)) == "depth_v3_stage2.pfm"
    assert os.path.basename(art.planes_path(d, 0, 1)) == "planes_v0_stage1.txt"
    assert os.path.basename(art.labels_path(d, 12)) == "labels_v12.png"
    assert os.path.basename(art.superpixels_path(d, 1)) == "superpixels_v1.txt"
    art.write_timings([("segment", 0, 12.5), ("refine", 1, 1234567.0)], os.path.join(d, "timings.tsv"))
    assert (tmp_path / "timings.tsv").read_text() == "stage\tview\tms\nsegment\t0\t12.5\nrefine\t1\t1.23457e+06\n"
    log = art.StatsLog(d)
    log.segment(0, 540)
    log.init(0, 32)
    log.close()
    log = art.StatsLog(d, resume=True)
    log.refine(0, 3)
    log.fuse(0, 0.25)
    log.close()
    assert (tmp_path / "stats.jsonl").read_text().splitlines() == [
        '{"stage":"segment","view":0,"superpixels":540}',
        '{"stage":"init","view":0,"levels":32}',
        '{"stage":"refine","view":0,"iterations":3}',
        '{"stage":"fuse","view":0,"epsilon":0.25}',
    ]


def _encode_filtered_png(path, img16, filters):
    """A 16-bit gray PNG whose row r uses PNG filter ``filters[r % len]`` (encoder per the PNG
    specification, independent of artifacts.py)."""
    import zlib
    h, w = img16.shape
    rows = img16.astype(">u2").view(np.uint8).reshape(h, 2 * w).astype(np.int64)
    bpp, out, prev = 2, [], np.zeros(2 * w, np.int64)
    for y in range(h):
        ft, cur = filters[y % len(filters)], rows[y]
        a = np.concatenate([np.zeros(bpp, np.int64), cur[:-bpp]])
        c = np.concatenate([np.zeros(bpp, np.int64), prev[:-bpp]])
        b = prev
        if ft == 0:
            pred = np.zeros_like(cur)
        elif ft == 1:
            pred = a
        elif ft == 2:
            pred = b
        elif ft == 3:
            pred = (a + b) >> 1
        else:
            p = a + b - c
            pa, pb, pc = np.abs(p - a), np.abs(p - b), np.abs(p - c)
            pred = np.where((pa <= pb) & (pa <= pc), a, np.where(pb <= pc, b, c))
        out.append(bytes([ft]) + ((cur - pred) & 0xFF).astype(np.uint8).tobytes())
        prev = cur

    def chunk(tag, body):
        return struct.pack(">I", len(body)) + tag + body + struct.pack(">I", zlib.crc32(tag + body))

    with open(path, "wb") as f:
        f.write(b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 16, 0, 0, 0, 0))
                + chunk(b"IDAT", zlib.compress(b"".join(out))) + chunk(b"IEND", b""))


def test_label_png_reader_all_filter_types(tmp_path):
    rng = np.random.default_rng(11)
    img = rng.integers(0, 65536, (10, 13)).astype(np.uint16)
    p = tmp_path / "f.png"
    for filters in ([0], [1], [2], [3], [4], [0, 1, 2, 3, 4]):
        _encode_filtered_png(str(p), img, filters)
        back, w, h = art.read_label_png(str(p))
        assert (w, h) == (13, 10) and np.array_equal(back, img.reshape(-1).astype(np.int32)), filters


def test_pipeline_config_validation():
    from paper_1812_06856_b200.api import InvalidParams
    from paper_1812_06856_b200.run import STAGE_ORDER, PipelineConfig

    assert STAGE_ORDER == ("segment", "init", "refine", "fuse", "eval")  # pipeline.hpp:25-28
    PipelineConfig(out_dir="x").validate()
    for bad, match in ((PipelineConfig(), "output directory"), (PipelineConfig(out_dir="x", stages=[]), "no stages"),
                       (PipelineConfig(out_dir="x", stages=["fuse", "x"]), "unknown stage"),
                       (PipelineConfig(out_dir="x", dump_every=-1), "bad pipeline"),
                       (PipelineConfig(out_dir="x", fusion_epsilon=-0.1), "bad pipeline")):
        with pytest.raises(InvalidParams, match=match):
            bad.validate()


def test_hexfloat_matches_libstdcxx_ostream(tmp_path):
    """The reference writes planes with ``f << std::hexfloat << value`` (pipeline.hpp:150-152):
    compile exactly that with g++ and compare its bytes with artifacts.hexfloat, and read the
    libstdc++ output back through read_planes."""
    import shutil
    import subprocess

    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    src = tmp_path / "hexf.cpp"
    src.write_text(
        "#include <cstdio>\n#include <iostream>\n#include <sstream>\n#include <vector>\n"
        "int main(){ std::vector<double> v; double x; while (std::fread(&x, 8, 1, stdin) == 1) v.push_back(x);\n"
        "  std::cout << v.size() / 4 << \"\\n\"; std::cout << std::hexfloat;\n"
        "  for (size_t i = 0; i + 3 < v.size(); i += 4)\n"
        "    std::cout << v[i] << \" \" << v[i+1] << \" \" << v[i+2] << \" \" << v[i+3] << \"\\n\";\n"
        "  return 0; }\n")
    exe = tmp_path / "hexf"
    subprocess.run(["g++", "-O1", "-o", str(exe), str(src)], check=True)
    rng = np.random.default_rng(13)
    vals = np.array(_doubles(rng, 400)[:4 * 200], np.float64)
    vals = vals[: len(vals) // 4 * 4]
    out = subprocess.run([str(exe)], input=vals.tobytes(), capture_output=True, check=True).stdout.decode()
    p = tmp_path / "planes.txt"
    art.write_planes(vals.reshape(-1, 4), str(p))
    assert p.read_text() == out
    p.write_text(out)
    assert art.read_planes(str(p)).tobytes() == vals.tobytes()

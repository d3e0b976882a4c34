"""Run artefacts of the reference pipeline, byte-compatible on disk.

Host-side file formats only — nothing here touches the GPU.  Each writer produces the bytes the
reference's writer produces (the label PNG: the same decoded pixels; PNG compression is an
encoder choice), and each reader accepts what the reference's writer emits, so a run directory
can be resumed by either implementation:

* ``write_pfm`` / ``read_pfm``            — io.hpp:67-111 (grayscale "Pf", rows bottom-up,
  native little-endian, scale "-1.0"; the reader byte-swaps big-endian files and rejects "PF",
  malformed headers, truncation and non-finite values);
* ``write_planes`` / ``read_planes``      — pipeline.hpp:145-172 (count line, then
  ``depth nx ny nz`` in C++ ``std::hexfloat`` = glibc ``%a``; parsed as strtod would);
* ``write_label_png`` / ``read_label_png`` — io.hpp:161-185 (16-bit single-channel PNG; labels
  outside [0, 65535] are an InvariantError; any other PNG type is a ParseError);
* ``write_depth_png``                     — io.hpp:116-135 (8-bit inverse depth, near = bright);
* ``write_superpixel_stats``              — pipeline.hpp:174-183 (``%.9g`` columns);
* ``write_timings`` / ``StatsLog``        — pipeline.hpp:252-256, 495-497 (``timings.tsv``,
  ``stats.jsonl``);
* ``depth_path`` / ``planes_path`` / ``labels_path`` / ``superpixels_path`` — the run-directory
  names of pipeline.hpp:139-143, 279-322, 350.
"""
from __future__ import annotations

import math
import os
import struct
import sys
import zlib
from typing import Iterable, List, Sequence, Tuple

import numpy as np


class IoError(RuntimeError):  # io.hpp IoError
    pass


class ParseError(RuntimeError):  # io.hpp ParseError
    pass


class InvariantError(RuntimeError):  # geometry.hpp InvariantError
    pass


# ------------------------------------------------------------------ run-directory names --

def view_tag(v: int) -> str:  # pipeline.hpp:139
    return "v%d" % v


def depth_path(run_dir: str, view: int, stage: int) -> str:  # pipeline.hpp:141-143
    return os.path.join(run_dir, "depth_%s_stage%d.pfm" % (view_tag(view), stage))


def planes_path(run_dir: str, view: int, stage: int) -> str:  # pipeline.hpp:310, 350
    return os.path.join(run_dir, "planes_%s_stage%d.txt" % (view_tag(view), stage))


def labels_path(run_dir: str, view: int) -> str:  # pipeline.hpp:279
    return os.path.join(run_dir, "labels_%s.png" % view_tag(view))


def superpixels_path(run_dir: str, view: int) -> str:  # pipeline.hpp:292-293
    return os.path.join(run_dir, "superpixels_%s.txt" % view_tag(view))


# ------------------------------------------------------------------------------- PFM --

def write_pfm(depth: np.ndarray, path: str) -> None:
    """io.hpp:67-78: "Pf\\n<w> <h>\\n-1.0\\n" (native little-endian), rows bottom-up."""
    d = np.ascontiguousarray(depth, dtype=np.float32)
    if d.ndim != 2:
        raise InvariantError("depth map must be 2-D")
    h, w = d.shape
    little = sys.byteorder == "little"
    try:
        with open(path, "wb") as f:
            f.write(b"Pf\n%d %d\n%s\n" % (w, h, b"-1.0" if little else b"1.0"))
            f.write(d[::-1].tobytes())
    except OSError as e:
        raise IoError("cannot open for writing: " + path) from e


def read_pfm(path: str) -> np.ndarray:
    """io.hpp:80-111.  Header tokens are whitespace-separated (``operator>>``); exactly one
    whitespace byte follows the scale."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError("cannot open: " + path) from e
    pos = 0

    def token() -> bytes:
        nonlocal pos
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        return data[start:pos]

    magic = token()
    if magic == b"PF":
        raise ParseError("expected grayscale Pf, got color PF: " + path)
    if magic != b"Pf":
        raise ParseError("not a PFM file: " + path)
    try:
        w, h, scale = int(token()), int(token()), float(token())
    except ValueError:
        raise ParseError("malformed PFM header: " + path) from None
    if w <= 0 or h <= 0 or scale == 0:
        raise ParseError("malformed PFM header: " + path)
    pos += 1  # f.get(): the single whitespace after the header
    n = w * h * 4
    if len(data) - pos < n:
        raise ParseError("truncated PFM data: " + path)
    dt = np.dtype("<f4") if scale < 0 else np.dtype(">f4")
    out = np.frombuffer(data, dtype=dt, count=w * h, offset=pos).astype(np.float32)
    out = out.reshape(h, w)[::-1].copy()
    if not np.isfinite(out).all():
        raise ParseError("non-finite value in PFM: " + path)
    return out


# ----------------------------------------------------------------------- hexfloat planes --

def hexfloat(x: float) -> str:
    """C++ ``std::hexfloat`` output of a double = glibc ``printf("%a")``: Python's
    ``float.hex`` with the mantissa's trailing zeros (and a bare '.') stripped."""
    x = float(x)
    if math.isnan(x):
        return "-nan" if math.copysign(1.0, x) < 0 else "nan"
    if math.isinf(x):
        return "-inf" if x < 0 else "inf"
    s = x.hex()  # [-]0x{0,1}.{13 hex}p{+,-}{exp}
    mant, exp = s.split("p")
    if "." in mant:
        head, frac = mant.split(".")
        frac = frac.rstrip("0")
        mant = head + ("." + frac if frac else "")
    if x == 0.0:
        exp = "+0"
    return mant + "p" + exp


def _strtod(tok: str) -> float:
    """strtod on one token: decimal, hexfloat, inf/nan (the reference ignores the end pointer,
    so an unparsable token yields 0.0)."""
    t = tok.strip()
    low = t.lower().lstrip("+-")
    neg = t.startswith("-")
    try:
        if low.startswith("0x"):
            return float.fromhex(t)
        if low in ("inf", "infinity"):
            return -math.inf if neg else math.inf
        if low.startswith("nan"):
            return math.nan
        return float(t)
    except ValueError:
        return 0.0


def write_planes(planes: np.ndarray, path: str) -> None:
    """pipeline.hpp:146-154: ``planes`` is f64[n, 4] = (depth, nx, ny, nz) per superpixel."""
    p = np.asarray(planes, dtype=np.float64).reshape(-1, 4)
    lines = ["%d\n" % p.shape[0]]
    lines.extend(" ".join(hexfloat(v) for v in row) + "\n" for row in p.tolist())
    try:
        with open(path, "w") as f:
            f.write("".join(lines))
    except OSError as e:
        raise IoError("cannot write " + path) from e


def read_planes(path: str) -> np.ndarray:
    """pipeline.hpp:156-172 -> f64[n, 4]."""
    try:
        with open(path, "r") as f:
            toks = f.read().split()
    except OSError as e:
        raise IoError("cannot open " + path) from e
    if not toks:
        return np.zeros((0, 4), np.float64)
    try:
        n = int(toks[0])
    except ValueError:
        n = 0  # `f >> n` failing leaves n = 0 in the reference
    if n < 0:
        raise ParseError("malformed plane count: " + path)
    if len(toks) - 1 < 4 * n:
        raise ParseError("truncated plane file: " + path)
    vals = [_strtod(t) for t in toks[1:1 + 4 * n]]
    return np.asarray(vals, dtype=np.float64).reshape(n, 4)


# ------------------------------------------------------------------------------- PNG --

_PNG_SIG = b"\x89PNG\r\n\x1a\n"


def _chunk(tag: bytes, body: bytes) -> bytes:
    return struct.pack(">I", len(body)) + tag + body + struct.pack(">I", zlib.crc32(tag + body) & 0xFFFFFFFF)


def _write_png(path: str, pixels: np.ndarray, bit_depth: int, color_type: int) -> None:
    h, w = pixels.shape[:2]
    if bit_depth == 16:
        rows = pixels.astype(">u2").reshape(h, -1).view(np.uint8)
    else:
        rows = pixels.astype(np.uint8).reshape(h, -1)
    raw = np.concatenate([np.zeros((h, 1), np.uint8), rows], axis=1).tobytes()  # filter 0 per row
    ihdr = struct.pack(">IIBBBBB", w, h, bit_depth, color_type, 0, 0, 0)
    try:
        with open(path, "wb") as f:
            f.write(_PNG_SIG + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", zlib.compress(raw, 6))
                    + _chunk(b"IEND", b""))
    except OSError as e:
        raise IoError("cannot write PNG: " + path) from e


def _read_png(path: str) -> Tuple[np.ndarray, int, int]:
    """Decode a non-interlaced PNG -> (samples u8/u16 [h, w, channels], bit_depth, color_type)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError("cannot read PNG: " + path) from e
    if not data.startswith(_PNG_SIG):
        raise IoError("cannot read PNG: " + path)
    pos, idat, hdr = 8, [], None
    while pos + 8 <= len(data):
        (n,) = struct.unpack(">I", data[pos:pos + 4])
        tag, body = data[pos + 4:pos + 8], data[pos + 8:pos + 8 + n]
        pos += 12 + n
        if tag == b"IHDR":
            hdr = struct.unpack(">IIBBBBB", body)
        elif tag == b"IDAT":
            idat.append(body)
        elif tag == b"IEND":
            break
    if hdr is None:
        raise IoError("cannot read PNG: " + path)
    w, h, depth, ctype, _, _, interlace = hdr
    chans = {0: 1, 2: 3, 4: 2, 6: 4}.get(ctype)
    if chans is None or interlace != 0 or depth not in (8, 16):
        raise ParseError("label PNG must be 16-bit single channel: " + path)
    bpp = chans * depth // 8
    stride = w * bpp
    try:
        raw = np.frombuffer(zlib.decompress(b"".join(idat)), np.uint8)
    except zlib.error:
        raise IoError("cannot read PNG: " + path) from None
    if raw.size < h * (stride + 1):
        raise IoError("cannot read PNG: " + path)
    raw = raw[:h * (stride + 1)].reshape(h, stride + 1)
    out = np.zeros((h, stride), np.uint8)
    prev = np.zeros(stride, np.uint8)
    for y in range(h):
        ft, line = raw[y, 0], raw[y, 1:].copy()
        if ft == 1:  # sub: a running sum per byte lane of the pixel, mod 256
            lanes = line[:stride - stride % bpp].reshape(-1, bpp)
            line = (np.cumsum(lanes, axis=0, dtype=np.uint64) & 0xFF).astype(np.uint8).reshape(-1)
        elif ft == 2:  # up
            line = (line + prev).astype(np.uint8)
        elif ft in (3, 4):  # avg / paeth: byte-serial (left neighbour is the decoded byte)
            cur, up = line.tolist(), prev.tolist()
            for x in range(stride):
                a = cur[x - bpp] if x >= bpp else 0
                b = up[x]
                if ft == 3:
                    pred = (a + b) >> 1
                else:
                    c = up[x - bpp] if x >= bpp else 0
                    pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
                    pred = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
                cur[x] = (cur[x] + pred) & 0xFF
            line = np.asarray(cur, np.uint8)
        elif ft != 0:
            raise IoError("cannot read PNG: " + path)
        out[y] = line
        prev = line
    if depth == 16:
        samples = out.view(">u2").astype(np.uint16).reshape(h, w, chans)
    else:
        samples = out.reshape(h, w, chans)
    return samples, depth, ctype


def write_label_png(labels: np.ndarray, width: int, height: int, path: str) -> None:
    """io.hpp:161-171."""
    lab = np.asarray(labels).reshape(height, width)
    if lab.size and (lab.min() < 0 or lab.max() > 65535):
        raise InvariantError("label out of 16-bit range")
    _write_png(path, lab.astype(np.uint16), 16, 0)


def read_label_png(path: str) -> Tuple[np.ndarray, int, int]:
    """io.hpp:173-185 -> (labels i32[h*w] row-major, width, height)."""
    samples, depth, ctype = _read_png(path)
    if depth != 16 or ctype != 0:
        raise ParseError("label PNG must be 16-bit single channel: " + path)
    h, w = samples.shape[:2]
    return samples.reshape(-1).astype(np.int32), w, h


def write_depth_png(depth: np.ndarray, d_min: float, d_max: float, path: str) -> None:
    """io.hpp:116-135: t = (1/d - 1/dmax)/(1/dmin - 1/dmax) clamped, lround(255 t); d <= 0 -> 0."""
    if not (0 < d_min < d_max):  # DepthRange::validate
        raise InvariantError("invalid depth range")
    d = np.asarray(depth, dtype=np.float32)
    inv_lo, inv_hi = 1.0 / d_max, 1.0 / d_min
    with np.errstate(divide="ignore"):
        t = (1.0 / d.astype(np.float64) - inv_lo) / (inv_hi - inv_lo)
    t = np.clip(t, 0.0, 1.0) * 255.0
    px = np.floor(t + 0.5)  # lround: half away from zero (t >= 0)
    px = np.where(d <= 0, 0, px).astype(np.uint8)
    _write_png(path, px, 8, 0)


# ------------------------------------------------------------------- text / tsv / jsonl --

def write_superpixel_stats(records: np.ndarray, path: str) -> None:
    """pipeline.hpp:174-183.  ``records`` is the lfdg_sp_record structured array
    (``_native.RECORD_DTYPE``: cx, cy, mean_color[3], pixel_count, gx, gy), id = row index."""
    lines = ["# id gx gy cx cy L a b count\n"]
    for i, r in enumerate(records):
        c = [float(np.float32(v)) for v in r["mean_color"]]
        lines.append("%d %d %d %s %s %s %s %s %d\n" % (
            i, int(r["gx"]), int(r["gy"]), "%.9g" % float(r["cx"]), "%.9g" % float(r["cy"]),
            "%.9g" % c[0], "%.9g" % c[1], "%.9g" % c[2], int(r["pixel_count"])))
    try:
        with open(path, "w") as f:
            f.write("".join(lines))
    except OSError as e:
        raise IoError("cannot write " + path) from e


def write_timings(timings: Iterable[Tuple[str, int, float]], path: str) -> None:
    """pipeline.hpp:495-497: header then ``stage\\tview\\tms`` with ostream's default %g."""
    with open(path, "w") as f:
        f.write("stage\tview\tms\n")
        for stage, view, ms in timings:
            f.write("%s\t%d\t%s\n" % (stage, view, "%g" % ms))


class StatsLog:
    """pipeline.hpp:252 (``stats.jsonl``, appended on resume) and the per-stage records."""

    def __init__(self, run_dir: str, resume: bool = False):
        self._f = open(os.path.join(run_dir, "stats.jsonl"), "a" if resume else "w")

    def segment(self, view: int, superpixels: int) -> None:  # pipeline.hpp:296-297
        self._f.write('{"stage":"segment","view":%d,"superpixels":%d}\n' % (view, superpixels))

    def init(self, view: int, levels: int) -> None:  # pipeline.hpp:333
        self._f.write('{"stage":"init","view":%d,"levels":%d}\n' % (view, levels))

    def refine(self, view: int, iterations: int) -> None:  # pipeline.hpp:392-393
        self._f.write('{"stage":"refine","view":%d,"iterations":%d}\n' % (view, iterations))

    def fuse(self, view: int, epsilon: float) -> None:  # pipeline.hpp:426
        self._f.write('{"stage":"fuse","view":%d,"epsilon":%s}\n' % (view, "%g" % epsilon))

    def eval(self, view: int, region: str, threshold: float, bad: float) -> None:  # pipeline.hpp:479-480
        self._f.write('{"stage":"eval","view":%d,"region":"%s","threshold":%s,"bad":%s}\n'
                      % (view, region, "%g" % threshold, "%g" % bad))

    def close(self) -> None:
        self._f.close()

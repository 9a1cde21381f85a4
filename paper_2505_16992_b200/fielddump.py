"""PFD1 field dumps of device fields (mirror of S/fielddump.py:1-159).

Same on-disk format as the reference (little-endian header b"PFD1", u32
version 1, u8 scalar width 4 / 8, u8 dimension, u16 block count, f64 time;
per block d x u32 resolution + u32 components; C-order payload; u32 zlib
CRC32 of the payload), the same atomic write (temporary file + rename) and
the same read-side verification (magic, version, sizes, checksum).

What differs is where the data comes from: fields live in HBM as (d, n)
structure-of-arrays tensors.  The writer streams each block's
(resolution..., components) C-order bytes to the file in chunks staged
through one pinned host buffer (device -> pinned copy, then file write and
running CRC), so a C4 field (302 MB) never needs a second full host copy.
Slab domains write collectively: rank 0 writes the header and every rank's
owned planes in order (:func:`dump_state_slab`).
"""

import os
import struct
import tempfile
import zlib

import numpy as np
import torch

__all__ = ["write_fields", "read_fields", "dump_state", "load_state",
           "dump_state_slab", "DumpError"]

MAGIC = b"PFD1"
VERSION = 1
_HEADER = struct.Struct("<4sIBBHd")
_CHUNK = 8 << 20          # bytes per staged chunk


class DumpError(IOError):
    """Malformed, truncated or corrupted field dump."""


def _np_dtype(precision):
    if precision not in ("double", "single"):
        raise ValueError("precision must be 'double' or 'single'")
    return np.dtype("<f8" if precision == "double" else "<f4")


class _Sink:
    """File writer with a running CRC32 of the payload."""

    def __init__(self, fh):
        self.fh = fh
        self.crc = 0
        self.nbytes = 0

    def payload(self, buf):
        mv = memoryview(buf).cast("B")
        self.crc = zlib.crc32(mv, self.crc)
        self.fh.write(mv)
        self.nbytes += mv.nbytes


def _stream_block(sink, arr, dtype):
    """C-order bytes of one block (resolution..., components) in chunks.
    Device tensors go through a pinned staging buffer."""
    if torch.is_tensor(arr):
        t = arr.detach()
        if t.dtype != (torch.float64 if dtype.itemsize == 8
                       else torch.float32):
            t = t.to(torch.float64 if dtype.itemsize == 8 else torch.float32)
        flat = t.contiguous().reshape(-1)
        per = max(1, _CHUNK // dtype.itemsize)
        if flat.is_cuda:
            stage = torch.empty(min(per, flat.numel()), dtype=flat.dtype,
                                pin_memory=True)
            for off in range(0, flat.numel(), per):
                cnt = min(per, flat.numel() - off)
                stage[:cnt].copy_(flat[off:off + cnt])
                sink.payload(stage[:cnt].numpy().astype(dtype, copy=False))
        else:
            for off in range(0, flat.numel(), per):
                sink.payload(flat[off:off + per].numpy().astype(dtype,
                                                                copy=False))
        return
    a = np.ascontiguousarray(np.asarray(arr), dtype=dtype)
    sink.payload(a.reshape(-1))


def _shape_of(a):
    return tuple(int(s) for s in a.shape)


def write_fields(path, blocks, time=0.0, precision="double"):
    """Write per-block arrays (each shaped resolution + (components,)),
    NumPy arrays or torch tensors (host or device).  Returns the byte
    count written (S/fielddump.py:41-88)."""
    dtype = _np_dtype(precision)
    if not blocks:
        raise ValueError("refusing to write a dump with no blocks")
    shapes = [_shape_of(b) for b in blocks]
    dim = len(shapes[0]) - 1
    if dim < 1:
        raise ValueError("block arrays need shape resolution + (components,)")
    for s in shapes:
        if len(s) != dim + 1:
            raise ValueError("blocks disagree on dimensionality")
        if int(np.prod(s)) == 0:
            raise ValueError("refusing to write an empty block")
    head = _HEADER.pack(MAGIC, VERSION, dtype.itemsize, dim, len(blocks),
                        float(time))
    table = b"".join(struct.pack(f"<{dim + 1}I", *s) for s in shapes)
    directory = os.path.dirname(os.path.abspath(path)) or "."
    fd, tmp = tempfile.mkstemp(dir=directory, suffix=".tmp")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(head)
            fh.write(table)
            sink = _Sink(fh)
            for b in blocks:
                _stream_block(sink, b, dtype)
            fh.write(struct.pack("<I", sink.crc & 0xFFFFFFFF))
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
    return len(head) + len(table) + sink.nbytes + 4


def read_fields(path):
    """Read a dump back: (blocks, time, precision) with the stored
    precision kept (S/fielddump.py:91-126)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEADER.size + 4:
        raise DumpError(f"{path}: truncated header")
    magic, version, width, dim, nblocks, time = _HEADER.unpack_from(raw, 0)
    if magic != MAGIC:
        raise DumpError(f"{path}: not a field dump (bad magic)")
    if version != VERSION:
        raise DumpError(f"{path}: unsupported dump version {version}")
    if width not in (4, 8):
        raise DumpError(f"{path}: bad scalar width {width}")
    off = _HEADER.size
    shapes = []
    for _ in range(nblocks):
        need = 4 * (dim + 1)
        if off + need > len(raw):
            raise DumpError(f"{path}: truncated block table")
        shapes.append(struct.unpack_from(f"<{dim + 1}I", raw, off))
        off += need
    dtype = np.dtype("<f8" if width == 8 else "<f4")
    total = sum(int(np.prod(s)) for s in shapes) * width
    if off + total + 4 != len(raw):
        raise DumpError(f"{path}: payload size mismatch "
                        f"(expected {off + total + 4}, got {len(raw)})")
    payload = memoryview(raw)[off:off + total]
    (crc,) = struct.unpack_from("<I", raw, off + total)
    if crc != (zlib.crc32(payload) & 0xFFFFFFFF):
        raise DumpError(f"{path}: payload checksum mismatch")
    blocks, pos = [], 0
    for s in shapes:
        cnt = int(np.prod(s))
        blocks.append(np.frombuffer(payload, dtype=dtype, count=cnt,
                                    offset=pos).reshape(s).copy())
        pos += cnt * width
    return blocks, time, ("double" if width == 8 else "single")


def _block_views(domain, field):
    """Per-block (resolution..., components) views of a flat (n, c) / (n,)
    field (torch or NumPy)."""
    f = field
    if f.ndim == 1:
        f = f[:, None] if not torch.is_tensor(f) else f.unsqueeze(1)
    views = []
    for b, shape in enumerate(domain.block_shapes):
        lo, hi = int(domain.offsets[b]), int(domain.offsets[b + 1])
        views.append(f[lo:hi].reshape(tuple(shape) + (f.shape[1],)))
    return views


def dump_state(path, domain, field, time=0.0, precision="double"):
    """Write a flat (n, c) or (n,) cell field (NumPy, or a torch tensor on
    any device) as per-block arrays (S/fielddump.py:129-137)."""
    return write_fields(path, _block_views(domain, field), time=time,
                        precision=precision)


def load_state(path, domain, device=None):
    """Read a dump written by ``dump_state`` back into a flat (n, c) array
    (a torch tensor on ``device`` when given) with the stored precision
    (S/fielddump.py:140-159)."""
    blocks, time, precision = read_fields(path)
    if len(blocks) != len(domain.block_shapes):
        raise DumpError(f"{path}: dump has {len(blocks)} blocks, domain has "
                        f"{len(domain.block_shapes)}")
    for arr, shape in zip(blocks, domain.block_shapes):
        if arr.shape[:-1] != tuple(shape):
            raise DumpError(f"{path}: block resolution {arr.shape[:-1]} does "
                            f"not match domain block {tuple(shape)}")
    ncomp = blocks[0].shape[-1]
    out = np.concatenate([a.reshape(-1, ncomp) for a in blocks])
    if device is not None:
        return torch.as_tensor(out, device=device), time, precision
    return out, time, precision


def dump_state_slab(path, slab, field, time=0.0, precision="double",
                    group=None):
    """Collective dump of a slab-decomposed field (slab.SlabDomain): the
    file holds the GLOBAL single-block channel, identical to ``dump_state``
    of the undecomposed field.  Rank 0 gathers the owned planes
    (torch.distributed, any backend) and writes."""
    import torch.distributed as dist
    own = slab.owned(field)
    if own.ndim == 1:
        own = own.unsqueeze(1)
    own = own.detach().to("cpu", torch.float64).contiguous()
    parts = [None] * slab.world
    dist.all_gather_object(parts, own, group=group)
    n = 0
    if dist.get_rank(group) == 0:
        full = torch.cat(parts, 0)
        n = write_fields(path, [full.reshape(tuple(slab.global_shape)
                                             + (full.shape[1],))],
                         time=time, precision=precision)
    dist.barrier(group=group)
    return n

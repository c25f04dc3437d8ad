"""Binary-format error types and atomic writes (sldlag/fileio.py:1-84).

The SLDM / SLDV / SLDQ readers and writers themselves are native
(csrc/sld_fileio.cpp); this module maps their status codes to the
reference's exception hierarchy so callers catch the same types.
"""
import os
import tempfile

from . import _native as N


class FormatError(Exception):
    """Base class for file-format problems (fileio.py:9-10)."""


class BadMagic(FormatError):
    """File does not start with the expected magic bytes (fileio.py:13-14)."""


class TruncatedFile(FormatError):
    """File ended before a complete record could be read (fileio.py:17-18)."""


def check_io(rc):
    """Raise the reference's exception for a file-format status code."""
    if rc == N.SLD_OK:
        return
    msg = N.load().sld_last_error().decode(errors="replace")
    if rc == N.SLD_E_MAGIC:
        raise BadMagic(msg)
    if rc == N.SLD_E_TRUNC:
        raise TruncatedFile(msg)
    if rc == N.SLD_E_FORMAT:
        raise FormatError(msg)
    N.check(rc)


def atomic_write(path, data: bytes):
    """Write via a temp file in the same directory and rename into place
    (fileio.py:66-84)."""
    path = os.fspath(path)
    d = os.path.dirname(path) or "."
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".tmp-", suffix=os.path.basename(path))
    try:
        with os.fdopen(fd, "wb") as f:
            f.write(data)
            f.flush()
            os.fsync(f.fileno())
        os.replace(tmp, path)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise

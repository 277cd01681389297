"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference HDG element-local
path (arXiv 1305.1489, /root/reference/proj). Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s cpu_baseline leg may import this package, and only as the
checker / CPU baseline. The product (`paper_1305_1489_b200`) never imports it.

Parity pinning: the reference C++ library cannot be compiled in this image
(Eigen3 and the doctest/CLI11 vendor headers are absent), so this restatement is
pinned by the reference's own known-answer tests and README golden errors,
ported in tests/test_oracle_kats.py.
"""
import os
import subprocess
import sys

_here = os.path.dirname(os.path.abspath(__file__))


def build(quiet: bool = True) -> None:
    """Compile the oracle extension in place (make -C oracle)."""
    out = subprocess.run(["make", "-C", _here, f"PY={sys.executable}"],
                         capture_output=quiet, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + (out.stdout or "") + (out.stderr or ""))


if os.environ.get("HDG_ORACLE_NATIVE") == "1":
    # CPU baseline: the same sources compiled -O3 -march=native for this host
    # (make native -> oracle/_native/); falls back to the portable build.
    _nat = os.path.join(_here, "_native")
    _out = subprocess.run(["make", "-C", _here, "native", f"PY={sys.executable}"], capture_output=True, text=True)
    NATIVE = _out.returncode == 0
    if NATIVE and _nat not in sys.path:
        sys.path.insert(0, _nat)
else:
    NATIVE = False
if _here not in sys.path:
    sys.path.insert(len(sys.path) if NATIVE else 0, _here)
try:
    import _hdg_oracle as core  # noqa: E402
except ImportError:  # built lazily in a fresh checkout
    build()
    import _hdg_oracle as core  # noqa: E402

__all__ = ["core", "build", "NATIVE"]

"""Recipe: install the UNMODIFIED reference (`prefillsim`, pure Python) into
oracle/_ref — TEST/BENCH INFRASTRUCTURE ONLY.

The reference is a setuptools package (/root/reference/pkg/pyproject.toml).
It is built by its own packaging from a scratch copy (the mounted tree is
read-only) with the offline toolchain:

    pip install --no-index --no-deps --no-build-isolation --target oracle/_ref <copy of /root/reference/pkg>

oracle/_ref is git-ignored (no reference source enters the history) but not
gpurun-ignored, so the installed package travels to the GPU box, where
bench.py's CPU legs (`--impl reference` and the GPU line's `cpu_baseline`)
import it and time the reference's own delta_for_rows /
compute_position_mask.  Nothing on the product path imports it.

`__graft_entry__.build()` runs this whenever /root/reference is mounted.
"""

from __future__ import annotations

import hashlib
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
DEST = ROOT / "oracle" / "_ref"
SRC = Path("/root/reference/pkg")
FILES = ("adapters.py", "model.py", "linalg.py", "errors.py", "workload.py", "costmodel.py")


def source_digest(pkg_dir: Path) -> str:
    h = hashlib.sha256()
    for name in FILES:
        p = pkg_dir / name
        if p.exists():
            h.update(p.read_bytes())
    return h.hexdigest()


def build(force: bool = False) -> Path | None:
    """Install prefillsim into oracle/_ref; None when the reference is not mounted."""
    if not (SRC / "pyproject.toml").exists():
        return DEST if (DEST / "prefillsim").exists() else None
    digest = source_digest(SRC / "src" / "prefillsim")
    stamp = DEST / "REF_SOURCE.txt"
    if not force and stamp.exists() and digest in stamp.read_text():
        return DEST
    with tempfile.TemporaryDirectory() as tmp:
        copy = Path(tmp) / "pkg"
        shutil.copytree(SRC, copy, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache"))
        if DEST.exists():
            shutil.rmtree(DEST)
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-deps", "--no-build-isolation",
                        "--quiet", "--target", str(DEST), str(copy)], check=True)
    stamp.write_text(f"prefillsim installed unmodified from {SRC}\nsha256({'+'.join(FILES)}) {digest}\n")
    return DEST


def import_reference():
    """(prefillsim.adapters, prefillsim.model) from oracle/_ref, or None."""
    if not (DEST / "prefillsim").exists():
        return None
    if str(DEST) not in sys.path:
        sys.path.insert(0, str(DEST))
    import prefillsim.adapters as RA
    import prefillsim.model as RM

    if not str(Path(RA.__file__).resolve()).startswith(str(DEST.resolve())):
        return None  # some other prefillsim shadows ours
    return RA, RM


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))

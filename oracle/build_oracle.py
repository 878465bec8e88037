"""Build the C restatement of the oracle (TEST INFRASTRUCTURE ONLY).

    python -m oracle.build_oracle

gcc -O3 -fopenmp, no fast-math and no FP contraction (products and sums are
rounded separately, as numpy does).  Output: oracle/_build/liboracle.so
(git-ignored, travels to the GPU box with the snapshot).
"""

from __future__ import annotations

import shutil
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "mdp_oracle.c"
OUT = HERE / "_build" / "liboracle.so"


def build(force: bool = False) -> Path:
    if not force and OUT.exists() and OUT.stat().st_mtime > max(SRC.stat().st_mtime,
                                                                Path(__file__).stat().st_mtime):
        return OUT
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        raise RuntimeError("gcc not found")
    OUT.parent.mkdir(exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [cc, "-O3", "-march=x86-64-v3", "-fopenmp", "-fno-fast-math", "-ffp-contract=off",
           "-shared", "-fPIC", str(SRC), "-o", str(tmp), "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stderr}")
    tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True))

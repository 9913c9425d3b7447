#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles the reference's own hot kernel
# (/root/reference/pkg/src/pcsir/_speedups.pyx, Cython, setup.py:19-30 flags -O3)
# where it lies, writing outputs only into oracle/_ref/. No reference source is
# copied into the repo; oracle/_ref/ is git-ignored and travels to the GPU box
# with the snapshot so bench.py --impl reference can time the reference kernel.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/pcsir/_speedups.pyx
OUT="$HERE/_ref"
[ -f "$SRC" ] || { echo "reference not present; skipping oracle/_ref"; exit 0; }
mkdir -p "$OUT"
python -m cython -3 -o "$OUT/_speedups.c" "$SRC"
PYINC=$(python -c 'import sysconfig; print(sysconfig.get_paths()["include"])')
NPINC=$(python -c 'import numpy; print(numpy.get_include())')
EXT=$(python -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')
gcc -O3 -fPIC -shared -I"$PYINC" -I"$NPINC" -o "$OUT/_speedups$EXT" "$OUT/_speedups.c"
echo "built $OUT/_speedups$EXT"

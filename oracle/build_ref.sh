#!/usr/bin/env bash
# Test infrastructure only (see oracle/README.md): compiles the reference's own
# compiled kernel core, /root/reference/pkg/src/adascale/_kernels.pyx, into
# oracle/_ref/ with the reference's own flags (pkg/setup.py:14-28:
# -O3 -ffp-contract=off -fopenmp).  Nothing from /root/reference is copied into
# tracked files: the generated C and the .so land in oracle/_ref/ (git-ignored).
#
# /usr/bin/gcc is used because the /opt/gcc wrapper cannot link -fopenmp
# ("cannot read spec file 'libgomp.spec'").
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${REF_ROOT:-/root/reference}/pkg/src/adascale/_kernels.pyx"
out="$here/_ref"
if [ ! -f "$src" ]; then
  echo "build_ref: $src not found (reference absent); keeping prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$out"
py="${PYTHON:-python3}"
ext="$($py -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
so="$out/_kernels$ext"
# the reference's UNMODIFIED Python package, staged next to its compiled core
# (git-ignored; travels to the GPU box) for the plugin-boundary test
# (tests/test_gpu_plugin.py: the reference's own solve_lp over the B200 table)
pkg="$(dirname "$src")"
mkdir -p "$out/pkg/adascale"
for f in "$pkg"/*.py; do
  [ "$out/pkg/adascale/$(basename "$f")" -nt "$f" ] || cp "$f" "$out/pkg/adascale/"
done
if [ -f "$so" ] && [ "$so" -nt "$src" ]; then
  exit 0
fi
"$py" -m cython -3 --module-name adascale._kernels "$src" -o "$out/_kernels.c"
inc_py="$($py -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
inc_np="$($py -c 'import numpy; print(numpy.get_include())')"
/usr/bin/gcc -shared -fPIC -O3 -ffp-contract=off -fopenmp \
  -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  -I"$inc_py" -I"$inc_np" "$out/_kernels.c" -o "$so.tmp" -fopenmp
mv "$so.tmp" "$so"
echo "build_ref: built $so"

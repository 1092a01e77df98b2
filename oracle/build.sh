#!/usr/bin/env bash
# Build the C oracle (always) and, when /root/reference is present, the
# reference's own Cython kernels into oracle/_ref/ (git-ignored; travels to the
# GPU box with the gpurun snapshot).  TEST INFRASTRUCTURE ONLY.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
gcc -O2 -ffp-contract=off -fPIC -shared -o "$here/liboracle.so" "$here/kernels_oracle.c"

ref_pyx=/root/reference/pkg/src/balsim/_kernels/_compiled.pyx
if [[ -f "$ref_pyx" ]]; then
    mkdir -p "$here/_ref"
    # cythonize the reference source where it lies; outputs only under _ref/
    cython -3 -o "$here/_ref/_compiled.c" "$ref_pyx"
    inc="$(python -c 'import sysconfig;print(sysconfig.get_paths()["include"])')"
    npinc="$(python -c 'import numpy;print(numpy.get_include())')"
    suffix="$(python -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')"
    gcc -O2 -fPIC -shared -I"$inc" -I"$npinc" \
        -o "$here/_ref/_compiled$suffix" "$here/_ref/_compiled.c"
fi

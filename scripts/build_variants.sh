# Build A/B variants of libmc.so into build_var/ (experiments only; the product build is _build.py).
# usage: bash scripts/build_variants.sh "name:-DFLAG=1 -DX=2" "name2:" ...
# Each variant is a full parallel build (_build.build with extra nvcc flags) into build_var/.
set -e
cd "$(dirname "$0")/.."
mkdir -p build_var
rm -f build_var/libmc_*.so
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  python - "$name" "$flags" <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2404_06359_b200 import _build
name, flags = sys.argv[1], sys.argv[2]
_build.build(force=True, lib=f"build_var/libmc_{name}.so", extra_flags=flags.split(), bdir=f"build_var/obj_{name}")
import shutil; shutil.rmtree(f"build_var/obj_{name}", ignore_errors=True)
print(" <-", name, flags)
PY
done

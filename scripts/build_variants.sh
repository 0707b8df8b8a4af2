# Build A/B variants of libmc.so into build_var/ (experiments only; the product build is _build.py).
# usage: bash scripts/build_variants.sh "name:-DFLAG=1 -DX=2" "name2=/path/to/decode.cu:" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p build_var
rm -f build_var/libmc_*.so
python -m paper_2404_06359_b200._build > /dev/null
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  src=paper_2404_06359_b200/csrc/decode.cu
  case "$name" in *=*) src="${name#*=}"; name="${name%%=*}";; esac
  if [ "$src" != paper_2404_06359_b200/csrc/decode.cu ]; then cp "$src" paper_2404_06359_b200/csrc/_variant.cu; src=paper_2404_06359_b200/csrc/_variant.cu; fi
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $flags \
       -c $src -o build_var/dec_$name.o 2>&1 \
       | grep -A2 "ILi2ELb0ELi7ELi3ELb1" | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '
  echo " <- $name ($flags)"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_var/libmc_$name.so \
       paper_2404_06359_b200/build/encode.o build_var/dec_$name.o -lpthread
  rm -f build_var/dec_$name.o paper_2404_06359_b200/csrc/_variant.cu
done

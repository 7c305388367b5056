#!/usr/bin/env bash
# Build an A/B variant of libmsk_b200.so into variants/<name>.so.
#   tools/build_variant.sh NAME [REV|-] [extra nvcc flags...]
# REV: git revision whose csrc/ to build ("-" = working tree).
set -euo pipefail
cd "$(dirname "$0")/.."
name=$1; rev=${2:--}; shift 2 || shift $#
src=paper_2603_29332_b200/csrc
tmp=paper_2603_29332_b200/_v_$name   # same depth as csrc/ so ../../include resolves
rm -rf "$tmp"; mkdir -p "$tmp"
if [ "$rev" = "-" ]; then
  cp $src/*.cu $src/*.cuh $src/*.cpp $src/*.hpp "$tmp"/
else
  for f in $(git ls-tree --name-only "$rev" $src/); do git show "$rev:$f" > "$tmp/$(basename "$f")"; done
fi
mkdir -p variants
JSON_INC=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
ARCH="-gencode arch=compute_100a,code=sm_100a"
objs=()
for f in "$tmp"/*.cu; do
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$JSON_INC -Iinclude "$@" -c "$f" -o "${f%.cu}.o"
  objs+=("${f%.cu}.o")
done
defs=(); for a in "$@"; do case "$a" in -D*) defs+=("$a");; esac; done  # -D flags also reach the host TU
g++ -std=c++17 -O2 -fPIC -I$JSON_INC "${defs[@]}" -c "$tmp/model.cpp" -o "$tmp/model_cpp.o"
nvcc $ARCH -shared -o variants/$name.so "${objs[@]}" "$tmp/model_cpp.o" -lcudart -ldl
rm -rf "$tmp"
echo "built variants/$name.so"

#!/bin/bash
# Build libepd.so with extra nvcc flags into ab/<name>.so (experiments only).
# usage: tools/build_variant.sh <name> [nvcc flags...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
obj=build/obj_$name
rm -rf "$obj"; mkdir -p "$obj" ab
pids=()
for f in paper_2501_05460_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -diag-suppress 177 "$@" \
    -c "$f" -o "$obj/$(basename "${f%.cu}").o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "ab/$name.so" "$obj"/*.o
echo "ab/$name.so"

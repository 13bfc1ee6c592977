#!/bin/bash
# Build libfgattn.so of a git revision into build/variants/<name>/ (A/B against the working tree).
#   scripts/build_rev.sh <rev> <name> [extra nvcc flags...]
set -e
rev=$1; name=$2; shift 2
dir=build/variants/$name
rm -rf "$dir" && mkdir -p "$dir/src"
git archive "$rev" paper_2509_16518_b200/csrc include | tar -x -C "$dir/src"
objs=()
for f in "$dir"/src/paper_2509_16518_b200/csrc/*.cu; do
  o="$dir/$(basename "${f%.cu}").o"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
    -I "$dir/src/include" "$@" -c "$f" -o "$o" &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$dir/lib$name.so" "${objs[@]}"
echo "$dir/lib$name.so"

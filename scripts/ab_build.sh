# Build a variant of libmp_b200.so from the current csrc into build/ab/<name>.so
# (development A/B timing; extra nvcc flags after the name).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
  "$@" -o build/ab/$name.so paper_2103_14695_b200/csrc/*.cu

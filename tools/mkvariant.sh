# usage: bash tools/mkvariant.sh NAME [-DMACRO=V ...]  -> tools/variants/libsar_NAME.so (tuning builds)
name=$1; shift
mkdir -p tools/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  -Xptxas -v -shared -cudart static -I include "$@" -o tools/variants/libsar_$name.so paper_2306_09784_b200/csrc/*.cu \
  2>&1 | grep -A2 "bp_kernelILb0ELb0ELb0ELi8ELi4E" | grep -E "registers|spill" | head -2

# Build an A/B variant of libefgp.so: one source file recompiled with extra -D flags, linked with the
# in-tree objects of the rest.  bash tools/build_variant.sh <out.so> <src.cu> [-DFOO=1 ...]
set -e
OUT=$1; SRC=$2; shift 2
O=paper_2210_10210_b200/build_obj
B=$(basename $SRC .cu)
TMP=$(mktemp /tmp/var_XXXX.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr \
  -I include -I paper_2210_10210_b200/csrc "$@" -c $SRC -o $TMP
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $(ls $O/*.o | grep -v "/$B.o") $TMP \
  -L/usr/local/cuda/lib64 -lcufft -lcusolver -ldl -Xlinker -rpath=/usr/local/cuda/lib64
rm -f $TMP

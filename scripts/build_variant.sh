# Build a variant of libblobtree_b200.so with extra nvcc flags for A/B timing
# (scripts/ab_march.sh).  usage: bash scripts/build_variant.sh <A|B|...> "<-DFLAG=1 ...>"
set -e
NAME=$1; EXTRA=$2
OBJ=build/var_$NAME
mkdir -p $OBJ paper_2304_09673_b200/lib/ab
NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $EXTRA"
for f in capi k_frame k_tile k_views k_tree k_compile k_trace k_util; do
  $NV -c paper_2304_09673_b200/csrc/$f.cu -o $OBJ/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2304_09673_b200/lib/ab/lib$NAME.so $OBJ/*.o build/obj/host/*.o \
  -Xlinker -soname,libblobtree_b200.so -lpthread -ldl -lrt
echo built paper_2304_09673_b200/lib/ab/lib$NAME.so

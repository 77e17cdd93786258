# Build a kernel variant library: mkvar.sh NAME SRC.cu "EXTRA NVCC FLAGS"
# -> tools/var/lib_NAME.so (the in-tree objects, SRC recompiled with the flags)
set -e
NAME=$1; SRC=$2; FLAGS=$3
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
C=$ROOT/paper_1902_08112_b200/csrc
make -C $C -s
T=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $FLAGS \
  -c $C/$SRC -o $T/${SRC%.cu}.o
OBJS=""
for o in $C/build/*.o; do b=$(basename $o); if [ "$b" = "${SRC%.cu}.o" ]; then OBJS="$OBJS $T/$b"; else OBJS="$OBJS $o"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared --cudart static -o $ROOT/tools/var/lib_$NAME.so $OBJS
rm -rf $T
echo built tools/var/lib_$NAME.so

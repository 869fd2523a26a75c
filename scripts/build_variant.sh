# Build an alternative library: one object (EXCL, e.g. l2p) replaced by SRC
# compiled with extra flags, linked with the current objects.
#   scripts/build_variant.sh NAME EXCL SRC.cu [nvcc flags...]
#     -> paper_2111_00110_b200/build_ab/lib_NAME.so
set -e
NAME=$1; EXCL=$2; SRC=$3; shift 3
D=paper_2111_00110_b200
mkdir -p $D/build_ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Iinclude -I$D/csrc "$@" -c $SRC -o $D/build_ab/${EXCL}_$NAME.o
OBJS=$(ls $D/build_obj/*.o | grep -v "/${EXCL}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/build_ab/lib_$NAME.so $OBJS $D/build_ab/${EXCL}_$NAME.o -lcudart
echo $D/build_ab/lib_$NAME.so

# Build an A/B variant of libmoe_b200.so with extra nvcc defines:
#   bash benchmarks/build_variant.sh NAME "-DFOO=1 -DBAR=0"
# -> exp/NAME/libmoe_b200.so (use with MOE_B200_LIB=exp/NAME/libmoe_b200.so)
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $ROOT/exp/$NAME
make -s -j8 -C $ROOT/paper_2205_10034_b200/csrc OUT=$ROOT/exp/$NAME/libmoe_b200.so \
  OBJDIR=$ROOT/exp/$NAME/build EXTRA_NVFLAGS="$FLAGS" $ROOT/exp/$NAME/libmoe_b200.so

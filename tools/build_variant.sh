# Build a variant of the native library with extra nvcc defines for A/B timing:
#   bash tools/build_variant.sh NAME -DFOO=1 ...   -> tools/_ab/NAME.so (load with EB_LIB_PATH)
NAME="$1"; shift
OUT=build_ab/$NAME; mkdir -p $OUT tools/_ab
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Iinclude -Ipaper_2003_01538_b200/csrc $*"
for f in conv_umma.cu block1.cu stem_pool.cu pointwise.cu combine.cu ref32.cu runtime.cu; do
  /usr/local/cuda/bin/nvcc $FLAGS -c paper_2003_01538_b200/csrc/$f -o $OUT/$f.o &
done
for f in tmap.cpp wire_decode.cpp; do
  /usr/local/cuda/bin/nvcc $FLAGS -x cu -c paper_2003_01538_b200/csrc/$f -o $OUT/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/_ab/$NAME.so $OUT/*.o
echo tools/_ab/$NAME.so

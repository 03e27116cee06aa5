# Build a library variant: one translation unit recompiled with extra flags, linked with the
# current objects of the others -> paper_1802_07844_b200/libhs_NAME.so (picked up by tools/ab.sh).
# Usage: bash tools/variant.sh NAME file.cu "-DFOO=1 ..."
set -e
cd "$(dirname "$0")/../paper_1802_07844_b200/csrc"
name=$1; src=$2; flags=$3
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
  --expt-relaxed-constexpr $flags -c $src -o variants/${name}_${src%.cu}.o 2> variants/${name}.ptxas.log
objs=""
for f in api plan sort cell_list pair gridding kspace fft; do
  if [ "$f.cu" = "$src" ]; then objs="$objs variants/${name}_$f.o"; else objs="$objs $f.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libhs_$name.so $objs -lcufft -lcudart
echo built ../libhs_$name.so

# Build variants of iga_tile.cu (macro flags) linked with the other objects of the current
# build: bash tools/tile_variants.sh "NAME:-DFLAG ..." ...; each lands in tune/NAME/libiga_b200.so
set -e
C=paper_2207_00280_b200/csrc
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -ccbin /usr/bin/g++"
OBJS=$(ls build/iga/*.o | grep -v iga_tile.o)
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  mkdir -p tune/$name
  ( $NV $flags -Xptxas -v -c -o tune/$name/iga_tile.o $C/iga_tile.cu > tune/$name/ptxas.log 2>&1 &&
    $NV -shared -o tune/$name/libiga_b200.so tune/$name/iga_tile.o $OBJS -lcudart ) &
done
wait
for v in "$@"; do name=${v%%:*}; test -f tune/$name/libiga_b200.so || { echo "variant $name failed:"; grep -m5 error tune/$name/ptxas.log; exit 1; }; done

# build + time k_gsf3_p3 variants (tools/p3_time.cu); usage: bash tools/p3_variants.sh "NAME:-DFLAGS" ...
set -e
mkdir -p build/p3
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo \
    -DVARIANT="\"$name\"" $flags -o build/p3/$name ${SRC:-tools/p3_time.cu} -Xptxas -v > build/p3/$name.log 2>&1 &
done
wait
for v in "$@"; do name=${v%%:*}; grep -A1 "k_gsf3_p3" build/p3/$name.log | grep -o "Used [0-9]* registers" | head -1 | sed "s/^/$name /"; done

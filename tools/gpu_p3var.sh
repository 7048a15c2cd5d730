# time built p3 variants (build/p3 is gpurun-ignored, so variants are copied to tune/p3)
for v in "$@"; do timeout 30 ./tune/p3/$v; done

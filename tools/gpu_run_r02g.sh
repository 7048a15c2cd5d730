set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/zeroc tools/dmma_zeroc.cu && ./build/zeroc
bash tools/p3_variants.sh "base:" "nostore:-DP3_ABL_NOSTORE" "split2:-DP3_SPLIT=2" "split1:-DP3_SPLIT=1" "sonly:-DP3_ABL_NOA -DP3_ABL_NOB" "sonly_nostore:-DP3_ABL_NOA -DP3_ABL_NOB -DP3_ABL_NOSTORE" "aonly:-DP3_ABL_NOB -DP3_ABL_NOS" "bonly:-DP3_ABL_NOA -DP3_ABL_NOS" "nos:-DP3_ABL_NOS" "nwb4:-DP3_NWB=4 -DP3_NWS=8"
for v in base nostore split2 split1 sonly sonly_nostore aonly bonly nos nwb4; do ./build/p3/$v; done

bash tools/p3_variants.sh "base:" "sord:-DP3_SORD=1" "sord_sonly:-DP3_SORD=1 -DP3_ABL_NOA -DP3_ABL_NOB" "sonly:-DP3_ABL_NOA -DP3_ABL_NOB"
for v in base sord sord_sonly sonly base sord; do ./build/p3/$v; done

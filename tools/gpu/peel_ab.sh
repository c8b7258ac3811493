# usage: VARIANTS="tag1 tag2" SCALE=26 T=10 MODES=2 bash tools/gpu/peel_ab.sh
# -> gpurun_out/pab<SCALE>_m<MODES>_<tag>.log (tag "new" = the working-tree library)
mkdir -p gpurun_out
S=${SCALE:-26}; TT=${T:-10}; M=${MODES:-2}
P=gpurun_out/pab${S}_m${M%%:*}
timeout 600 python tools/peel_ab.py $S $TT $M > ${P}_new.log 2>&1
for v in $VARIANTS; do
  DG_B200_LIB=paper_2311_04333_b200/libdg_b200_$v.so timeout 600 python tools/peel_ab.py $S $TT $M > ${P}_$v.log 2>&1
done
timeout 600 python tools/peel_ab.py $S $TT $M >> ${P}_new.log 2>&1

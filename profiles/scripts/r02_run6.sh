bash profiles/scripts/ab.sh v6 profiles/variants/libtgs_vA.so profiles/variants/libtgs_vB.so profiles/variants/libtgs_vC.so profiles/variants/libtgs_vD.so env:TGS_EXACT=0 > gpurun_out/ab_v6.txt 2>&1

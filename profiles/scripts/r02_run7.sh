bash profiles/scripts/ab.sh v7 profiles/variants/libtgs_c68.so profiles/variants/libtgs_c78.so profiles/variants/libtgs_c58.so env:TGS_EXACT=0 > gpurun_out/ab_v7.txt 2>&1

# A/B of library builds (tools/_prof/lib_<X>.so) on the bench step; LIBS overrides the list
mkdir -p gpurun_out
timeout 1500 python tools/ab_multi.py --libs ${LIBS:-base,uni} --rounds ${ROUNDS:-2} > gpurun_out/ab_${TAG:-x}.log 2>&1

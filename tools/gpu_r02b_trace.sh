for v in "" SPIN; do for ab in 0 3; do A2D_PROF_VARIANT=$v A2D_TRACE=1 A2D_ABLATE=$ab timeout 300 python tools/bwd_prof.py > gpurun_out/r3_trace${v}_$ab.json 2>&1; echo v=$v ab=$ab rc=$?; done; done

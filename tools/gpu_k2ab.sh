mkdir -p gpurun_out
timeout 1200 python tools/k2_ab.py --config ${CFG:-c3} --batch ${BATCH:-256} "$@" > gpurun_out/k2ab.log 2>&1
cat gpurun_out/k2ab.log

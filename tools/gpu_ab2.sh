mkdir -p gpurun_out
GACQ_LIB=exp/libgacq_$1.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_$1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$1.log
shift 0
bash tools/gpu_ab.sh "$@"

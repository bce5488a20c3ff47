mkdir -p gpurun_out
GACQ_LIB=exp/libgacq_stock.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_stock.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stock.log
for v in dit stock; do GACQ_LIB=exp/libgacq_$v.so timeout 300 python bench.py --config g5 --steps 5 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/g5_$v.json 2>&1; done

# full GPU suite (+ optional extra pytest args), log to gpurun_out/pytest_gpu.log
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log

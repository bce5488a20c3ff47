# generic path: parity subset + G5/G8 timing (args: tag)
mkdir -p gpurun_out
T=${1:-gen}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or generic or power_of_two" > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
tail -5 gpurun_out/${T}_pytest.log
for cf in g5 g8; do timeout 600 python tools/k2_ab.py --config $cf --batch 64 default 2>&1 | cut -c1-250; done

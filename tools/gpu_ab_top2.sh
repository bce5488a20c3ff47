mkdir -p gpurun_out
(for cf in c3 c1 c4; do echo "== $cf"; timeout 600 python tools/k2_ab.py --config $cf --batch $([ $cf = c4 ] && echo 16 || echo 512) default old 2>&1 | cut -c1-400; done) > gpurun_out/ab_top2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -k "radius" tests/test_gpu_multirank.py -q -x > gpurun_out/pytest_radius.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_radius.log
cat gpurun_out/ab_top2.log; tail -5 gpurun_out/pytest_radius.log

# generic-path A/B: parity subset on the in-tree build, then G5/G8 correlation times of the
# in-tree build against exp/libgacq_<v>.so variants (tools/build_variant.sh): tools/gpu_gen_ab.sh v1 v2 ...
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_configs.py -q -x -k "generic or power_of_two or golden or random" > gpurun_out/pytest_gen.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gen.log; tail -2 gpurun_out/pytest_gen.log
for cf in g5 g8; do timeout 600 python tools/k2_ab.py --config $cf --batch 128 default "$@" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['variant'], d['corr_ms'], d['fwd_ms'], round(d['frac'], 4), d['rows'])
    else: print(l[:300])"; done

# A/B of K2 variants (exp/libgacq_<v>.so) against the in-tree build: tools/gpu_ab.sh "<configs>" v1 v2 ...
mkdir -p gpurun_out
CF=$1; shift
(for cf in $CF; do echo "== $cf"; timeout 900 python tools/k2_ab.py --config $cf --batch $([ $cf = c4 ] && echo 16 || echo 512) default "$@" 2>&1 | cut -c1-330; done) > gpurun_out/ab.log
cat gpurun_out/ab.log

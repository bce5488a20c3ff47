mkdir -p gpurun_out
for v in "$@"; do GACQ_LIB=exp/libgacq_$v.so timeout 300 python bench.py --config c4 --steps 5 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/c4_$v.json 2>&1; done

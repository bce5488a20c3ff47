# A/B of libgacq builds under exp/: bench C3 K1/K2 times per variant
mkdir -p gpurun_out
for v in "$@"; do
  GACQ_LIB=exp/libgacq_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/ab_$v.json 2>&1
done

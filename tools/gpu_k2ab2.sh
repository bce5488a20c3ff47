mkdir -p gpurun_out
for b in 64 256 1024; do
echo "batch $b"
timeout 900 python tools/k2_ab.py --config c3 --batch $b "$@" 2>&1 | cut -c1-200
done > gpurun_out/k2ab.log
cat gpurun_out/k2ab.log

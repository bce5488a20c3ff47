mkdir -p gpurun_out
python -c "
import paper_1309_0052_b200 as g
e=g.AcqEngine(4.092e6, list(range(1,33)), g.AcqConfig(noncoherent_rounds=10, doppler_min_hz=-5000, doppler_max_hz=5000, doppler_step_hz=500))
print(e.info)" > gpurun_out/info.txt 2>&1
for n in 3 2; do GACQ_CORR_CTAS_PER_SM=$n timeout 300 python bench.py --steps 10 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/bench_tc$n.json 2>&1; done

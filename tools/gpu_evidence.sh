# Round evidence: -m gpu suite, smoke, C3 bench line, reference arm, generic bench lines, launch list, K1/K2 ncu capture (args: tag)
mkdir -p gpurun_out
T=${1:-r02d}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log; tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
for c in g5 g8; do timeout 900 python bench.py --config $c --steps 10 --tracking-epochs 1 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gacq_ -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/${T}_b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gacq_(corr_pfa|fwd_pfa)" -s 2 -c 2 -o gpurun_out/${T}_prof -f python bench.py --steps 3 --warmup 3 --batch 64 --no-cpu-baseline --tracking-epochs 1 > gpurun_out/${T}_prof.log 2>&1
# (the generic-path capture is tools/gpu_prof_gen.sh: two --set full reports exceed what one gpurun call brings back, 64 MiB)
for f in gpurun_out/${T}_bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().splitlines()[-1])
    r = d.get("roofline") or {}
    print(f.split("/")[-1], round(d["value"] / 1e6, 3), "e2e", round(d["e2e"]["value"] / 1e6, 3), "frac", round(r.get("frac") or 0, 3), "clk", d.get("clocks"))
except Exception as e:
    print(f, "ERR", e)
PY
done

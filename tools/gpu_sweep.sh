# every config's bench line + the 2-rank launcher on one GPU (args: tag)
mkdir -p gpurun_out
T=${1:-r02}
for c in c1 c2 c4 c5 d8 g5 g8; do timeout 900 python bench.py --config $c --steps 10 --tracking-epochs 1 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --gpus 2 --device-map 0,0 --steps 10 --tracking-epochs 1 > gpurun_out/${T}_bench_c3_2ranks.json 2> gpurun_out/${T}_bench_c3_2ranks.err; echo "2ranks rc=$?"
for f in gpurun_out/${T}_bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().splitlines()[-1])
    r = d.get("roofline", {})
    print(f.split("/")[-1], round(d["value"] / 1e6, 3), "e2e", round(d["e2e"]["value"] / 1e6, 3), "frac", round(r.get("frac") or 0, 3),
          "cpu", round((d.get("cpu_baseline") or {}).get("value", 0) / 1e3, 2), "k", (d.get("cpu_baseline") or {}).get("decisions_vs_gpu"))
except Exception as e:
    print(f, "ERR", e)
PY
done

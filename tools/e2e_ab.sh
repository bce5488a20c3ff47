for v in default grow2 grow8 grow16; do
  if [ $v = default ]; then unset GACQ_LIB; else export GACQ_LIB=exp/libgacq_$v.so; fi
  for c in c3 c1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --tracking-epochs 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$v', '$c', round(d['value']/1e6,3), round(d['e2e']['value']/1e6,3), round(d['e2e_int8']['value']/1e6,3))"
  done
done

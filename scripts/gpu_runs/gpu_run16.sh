mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -3
run() { # name env...
  name=$1; shift
  env "$@" timeout 900 python scripts/auc_modes.py > gpurun_out/pol_$name.jsonl 2>&1
  echo "== $name"; grep '"mode"' gpurun_out/pol_$name.jsonl | python -c "
import sys,json
v=[json.loads(l) for l in sys.stdin]
import statistics as s
print(' '.join(f\"{x['mode']}:{x['aucroc']:.4f}/{x['embed_s']:.2f}s\" for x in v))
for m in sorted(set(x['mode'] for x in v)):
    a=[x['aucroc'] for x in v if x['mode']==m]; print(m, 'mean', round(s.mean(a),4), 'n', len(a))
"
}
run c1_d16 GB_INFLIGHT_DIV=16 GRAPH=c1 MODES=cap0 SEEDS=1,2,3,4,5,1,2,3
run c1_f256 GB_INFLIGHT_FLOOR=256 GRAPH=c1 MODES=cap0 SEEDS=1,2,3,4,5,1,2,3
run c1_d4f256 GB_INFLIGHT_DIV=4 GB_INFLIGHT_FLOOR=256 GRAPH=c1 MODES=cap0 SEEDS=1,2,3,4,5,1,2,3
run c1_tour GRAPH=c1 MODES=tour1,tour2,tour4 SEEDS=1,2,3,4,5
run c3_pol GRAPH=c3 MODES=cap0 SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000
run c3_d4 GB_INFLIGHT_DIV=4 GB_INFLIGHT_FLOOR=256 GRAPH=c3 MODES=cap0 SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000
run c3_d1 GB_INFLIGHT_DIV=1 GB_INFLIGHT_FLOOR=1024 GRAPH=c3 MODES=cap0 SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000

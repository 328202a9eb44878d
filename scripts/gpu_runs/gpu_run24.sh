mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
CAPS=64,256,1024 PASSES=200 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -3
GB_PIPE=1 DIM=32 V=500 CAPS=256 PASSES=2000 timeout 300 python scripts/profile_small_level.py 2>&1 | tail -1
UNIT=edge-scaled timeout 1200 python scripts/bench_multilevel.py c3 1000 > gpurun_out/ml_c3_es_pipe.jsonl 2>&1; grep -E "level|summary" gpurun_out/ml_c3_es_pipe.jsonl | cut -c1-200
GRAPH=c1 MODES=cap0 SEEDS=1,2,3,4,5,1,2,3 timeout 900 python scripts/auc_modes.py > gpurun_out/pol_c1_pipe.jsonl 2>&1; grep '"mode"' gpurun_out/pol_c1_pipe.jsonl | python -c "
import sys,json,statistics as s
v=[json.loads(l) for l in sys.stdin]; a=[x['aucroc'] for x in v]; print('c1 mean', round(s.mean(a),4), [round(x,4) for x in a], 'embed', round(s.mean([x['embed_s'] for x in v]),3))"
GRAPH=c3 MODES=cap0 SEEDS=1,2 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 900 python scripts/auc_modes.py 2>&1 | grep '"mode"'

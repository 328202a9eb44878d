timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
GRAPH=c3 MODES=cap0 SEEDS=1 UNIT=vertex-pass EPOCHS=100 EVAL_SAMPLE=1000000 timeout 900 python scripts/auc_modes.py 2>&1 | tail -2 | cut -c1-300

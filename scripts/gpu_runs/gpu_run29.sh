timeout 900 python -m pytest tests -q -m gpu -k "fidelity or zero_epochs or mismatch" 2>&1 | tail -5

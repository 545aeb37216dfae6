python -m pytest tests -q -m gpu -x --timeout 2400 2>&1 | tail -15

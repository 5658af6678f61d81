timeout 900 python -m pytest tests -q -x -m gpu --timeout 200 2>&1 | tail -2

python -m pytest tests -m gpu -q --maxfail=60 -p no:cacheprovider --deselect tests/test_wide.py 2>&1 | tail -40

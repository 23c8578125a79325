python tools/layout_probe.py
python tools/layout_probe.py
python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1

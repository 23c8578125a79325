python tools/layout_probe.py
python -m pytest tests/test_gpu.py -q -x -k "layout or dense or symm or tile_matrix or round_trip" -p no:cacheprovider 2>&1 | tail -2

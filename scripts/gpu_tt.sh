python scripts/tile_trace.py --config 5 --n 20000000 2>/dev/null
python scripts/tile_trace.py --config 3 --n 20000000 2>/dev/null

python scripts/tile_trace.py --config 2 --n 312500
python scripts/tile_trace.py --config 2 --n 2500000
python scripts/tile_trace.py --config 2 --n 10000000
python scripts/tile_trace.py --config 5 --n 20000000

timeout -s KILL 900 python -m pytest tests/test_gpu_selection.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout -s KILL 600 python scripts/kmeans_probe.py 2000
STGP_KMEANS_CERTIFIED=0 timeout -s KILL 900 python scripts/kmeans_probe.py 2000

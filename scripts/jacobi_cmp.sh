timeout 600 python -m pytest tests/test_reconstruction.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
RBG_JACOBI=elem timeout 600 python -m pytest tests/test_reconstruction.py -q -m gpu -p no:cacheprovider 2>&1 | tail -1
timeout 600 python scripts/next_kernels_probe.py 2>&1 | tail -3
RBG_JACOBI=elem timeout 600 python scripts/next_kernels_probe.py 2>&1 | tail -1

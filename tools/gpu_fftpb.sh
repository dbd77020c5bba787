for pb in 0 2 3 4 6 8 12; do echo "ADP_FFT_PB=$pb"; ADP_FFT_PB=$pb timeout 300 python tools/prof_fft.py; ADP_FFT_PB=$pb timeout 300 python tools/prof_fft_solve.py --iters 10 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_fft.py -m gpu -x -q 2>&1 | tail -3

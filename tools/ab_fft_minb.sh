# A/B of the FFT kernels' minimum-blocks-per-SM launch bounds (rebuilds fft.o on the box)
set -x
cd paper_2502_09758_b200/csrc
for v in "3 3" "2 3" "3 2" "2 2"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -Xptxas -v \
    -DFFT_COL_MINB=$1 -DFFT_ROW_MINB=$2 -c fft.cu -o build/fft.o > ../../gpurun_out/fft_ptxas_$1$2.log 2>&1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/libadpb200.so build/*.o
  (cd ../.. && timeout 300 python tools/prof_fft_solve.py > gpurun_out/fft_ab_$1$2.txt 2>&1)
done

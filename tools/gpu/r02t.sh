set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd tools/micro
./fp64mix > ../../gpurun_out/r02t_fp64mix.txt 2>&1
./stencilvar > ../../gpurun_out/r02t_stencilvar.txt 2>&1
cat ../../gpurun_out/r02t_fp64mix.txt ../../gpurun_out/r02t_stencilvar.txt

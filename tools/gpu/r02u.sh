set -x
cd tools/micro
./fp64mix > ../../gpurun_out/r02u_fp64mix.txt 2>&1
cat ../../gpurun_out/r02u_fp64mix.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:stage -s 403 -c 1 -o ../../gpurun_out/r02u_stencilvar_const ./stencilvar > ../../gpurun_out/r02u_ncu.log 2>&1; echo "ncu rc $?"
tail -3 ../../gpurun_out/r02u_ncu.log

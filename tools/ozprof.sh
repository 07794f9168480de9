# one ncu --set full capture of the Ozaki GEMM at ld=1024 with digit output
timeout 600 ncu --set full --import-source on -k regex:oz_gemm_kernel -c 1 -o gpurun_out/oz_gemm -f python tools/oz_check.py 1024 > gpurun_out/oz_ncu.log 2>&1

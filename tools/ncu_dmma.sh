python -c "import __graft_entry__ as g; g.build()" > /dev/null
for sh in "2048 768 256 1 1" "2048 1024 256 1 1" "2048 256 1024 1 1" "2048 256 256 1 1" "256 1024 2048 0 0"; do python tools/dmma_one.py $sh; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 1 -c 1 -o gpurun_out/dmma_qkv -f python tools/dmma_one.py 2048 768 256 1 1 > gpurun_out/ncu_dmma.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dmma -s 1 -c 1 -o gpurun_out/dmma_fc -f python tools/dmma_one.py 2048 1024 256 1 1 >> gpurun_out/ncu_dmma.log 2>&1
echo done

# ncu --set full captures of the secondary kernels: the Go1-shape step tail
# (loco_tail_kernel, 8192 worlds x 100 steps) and the pixel stack kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/exp_tail.py > gpurun_out/tail_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:loco_tail_kernel -s 1 -c 1 \
  -o gpurun_out/prof_tail -f python tools/exp_tail.py > gpurun_out/ncu_tail.log 2>&1
timeout 300 python tools/exp_pixstack.py 8192 > gpurun_out/pixstack_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pixel_stack_kernel -s 2 -c 1 \
  -o gpurun_out/prof_pixstack -f python tools/exp_pixstack.py 8192 > gpurun_out/ncu_pixstack.log 2>&1
echo done

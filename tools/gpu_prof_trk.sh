mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:gacq_epl -s 1 -c 1 -o gpurun_out/prof_trk -f python tools/trk_probe.py > gpurun_out/prof_trk.log 2>&1

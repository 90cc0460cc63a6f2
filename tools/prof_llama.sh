python tools/k2_subset.py llama3.2 1
python tools/k2_subset.py resnet152 1
python tools/k2_subset.py gpt2/ 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof/k_replay_llama python tools/k2_subset.py llama3.2 1 > /dev/null 2>&1
ls gpurun_out/prof/

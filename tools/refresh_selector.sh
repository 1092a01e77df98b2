# refresh the measured-latency selector profiles and the CP=4/8 single-GPU rank emulation (dev aid)
set -e
python -m paper_2503_17924_b200.calibrate --hq 32 --hkv 32 --d 128 --out gpurun_out/b200_llama7b_h32_d128.profile.json > gpurun_out/cal7b.log
python -m paper_2503_17924_b200.calibrate --hq 64 --hkv 8 --d 128 --out gpurun_out/b200_llama70b_h64_kv8_d128.profile.json > gpurun_out/cal70b.log
python tools/cp_emulate.py --window 131072 --cps 4 8 --profile gpurun_out/b200_llama7b_h32_d128.profile.json --out gpurun_out/cp_emulate_7b.json | tail -1
python tools/cp_emulate.py --window 131072 --cps 4 8 --hq 64 --hkv 8 --profile gpurun_out/b200_llama70b_h64_kv8_d128.profile.json --out gpurun_out/cp_emulate_70b.json | tail -1
python tools/config5.py --iters 4 --sample 6 --out gpurun_out/config5.json | cut -c1-400
bash tools/docsweep.sh | head -4

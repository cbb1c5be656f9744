export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "not full_size" > gpurun_out/t32.log 2>&1; echo "exit $?" >> gpurun_out/t32.log
timeout 900 python tools/bench_configs.py 3 5 > gpurun_out/configs32.jsonl 2>/dev/null
python tools/ncu_target.py > gpurun_out/ncus_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"stft_phat" --csv --log-file gpurun_out/stft_time.csv python tools/ncu_target.py > /dev/null 2>&1

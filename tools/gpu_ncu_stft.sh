export PYTHONPATH=$PWD
python tools/ncu_target.py > gpurun_out/ncus_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stft_phat" -s 1 -c 1 -o gpurun_out/prof_stft python tools/ncu_target.py > gpurun_out/ncus.log 2>&1
echo "exit $?" >> gpurun_out/ncus.log

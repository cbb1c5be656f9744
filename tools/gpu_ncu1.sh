export PYTHONPATH=$PWD
python tools/ncu_target.py > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|stft|finalize|zsplit" --csv --log-file gpurun_out/launches.csv python tools/ncu_target.py > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|stft_phat_kernel|finalize_kernel" -s 6 -c 5 -o gpurun_out/prof_r01 python tools/ncu_target.py > gpurun_out/ncu2.log 2>&1
echo "exit $?" >> gpurun_out/ncu2.log

export PYTHONPATH=$PWD
python tools/ncu_target.py > gpurun_out/ncuf_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|stft|finalize|zsplit" --csv --log-file gpurun_out/launches_final.csv python tools/ncu_target.py > gpurun_out/ncuf1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel|stft_phat|finalize|zsplit|gemm_kernel" -s 7 -c 6 -o gpurun_out/prof_final python tools/ncu_target.py > gpurun_out/ncuf2.log 2>&1
echo "exit $?" >> gpurun_out/ncuf2.log

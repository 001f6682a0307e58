for n in 148 96 64 32 16; do LLEP_GEMM_SMS=$n python tools/wgrad_bench.py small 5760 2880; done > gpurun_out/wgrad_sms.txt 2>&1
for n in 148 120 96; do LLEP_GEMM_SMS=$n python tools/wgrad_bench.py hot 5760 2880; done >> gpurun_out/wgrad_sms.txt 2>&1
python tools/wgrad_bench.py both 5760 2880 >> gpurun_out/wgrad_sms.txt 2>&1
cat gpurun_out/wgrad_sms.txt

cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "batched or prefill" 2>&1 | tail -2
bash abtmp/run.sh

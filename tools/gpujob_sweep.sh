bash tools/gpujob_stages.sh
python tests/gpu_p50.py C1 C2 C4

# full measurement round (run under gpurun): bench, reference arm, launch list, ncu capture, phases
tag=${1:-latest}
bash tests/profile_round.sh $tag
python tests/gpu_phases.py C2 1024 > gpurun_out/phases_c2_${tag}.txt 2>&1
python tests/gpu_phases.py C4 64 > gpurun_out/phases_c4_${tag}.txt 2>&1

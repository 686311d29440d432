# stage times of C2 x 1024, C4 x 64 and the C5 corpus (no phase timing)
SLOS_NO_PHASES=1 SLOS_SOLVES=4 python tests/gpu_phases.py C2 1024 2>&1 | tail -2
SLOS_NO_PHASES=1 SLOS_SOLVES=3 python tests/gpu_phases.py C4 64 2>&1 | tail -2
SLOS_NO_PHASES=1 SLOS_SOLVES=3 python tests/gpu_phases_c5.py 2>&1 | tail -2

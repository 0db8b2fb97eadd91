# per-phase stamps of the full 32-block F and B tasks (full grid, never mode) at HEAD
mkdir -p gpurun_out
timeout 300 python profiles/st_phases.py blocks=32 > gpurun_out/r7p_phases_fwd32.txt 2>&1
timeout 300 python profiles/st_phases.py blocks=32 bwd=1 > gpurun_out/r7p_phases_bwd32.txt 2>&1
tail -1 gpurun_out/r7p_phases_fwd32.txt gpurun_out/r7p_phases_bwd32.txt

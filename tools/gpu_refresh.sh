# Refresh of the committed evidence on one B200 (run under gpurun): ncu --set full captures of the
# operator kernels with their summaries, launch list, bench lines and smoke() first
# (tools/gpu_refresh_captures.sh), then the GPU suite, the reference arm, the 8-rank share-gpu line
# and the degree / workload sweeps (tools/gpu_refresh_suite.sh). The halves can run as two gpurun
# calls. Every ncu command follows a plain run of the same command that exited 0
# (B200_PROFILING.md). Copy gpurun_out/ncu_full_summary.json to profiles/ afterwards.
bash tools/gpu_refresh_captures.sh
bash tools/gpu_refresh_suite.sh

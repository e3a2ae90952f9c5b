# End-of-round evidence: GPU tests, smoke, the default bench line, ncu captures.
O=gpurun_out/${1:-r02g}; mkdir -p $O
bash tools/gpu_check.sh $(basename $O)
bash tools/profile_captures.sh $O

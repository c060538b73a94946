N=4 CONFIGS="c2 c3 c4 c5 c2x4 c3x4 c4w4 c5w4" TAG=_s14 bash scripts/gpu_state.sh
N=2 CONFIGS="c2 c3 c4 c5" TAG=_s14 CUDA_VISIBLE_DEVICES=0,1 bash scripts/gpu_state.sh

bash scripts/gpu_round.sh ncu
CASES="permute router decode prefill ep attention" timeout 2400 bash scripts/sanitize.sh

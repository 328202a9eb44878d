# round 2, run 37: C3 levels 0-3 (edge-scaled, 10 epochs each) under kernel
# layout variants: default, KIND 0 (GB_PASS_SMEM=0), 16 and 4 lanes per source
mkdir -p gpurun_out
for L in 0 1 2 3; do
for v in default smem0 lanes16 lanes4; do
unset GB_PASS_SMEM GB_GROUP_LANES
case $v in smem0) export GB_PASS_SMEM=0;; lanes16) export GB_GROUP_LANES=16;; lanes4) export GB_GROUP_LANES=4;; esac
LEVEL=$L EPOCHS=10 timeout 300 python scripts/profile_c3_levels.py 2>/dev/null | sed "s/^/{\"variant\": \"$v\", \"r\": /; s/\$/}/" >> gpurun_out/r2_37_levels_layout.jsonl
done; done

set -u
mkdir -p gpurun_out
bash scripts/gpu_prof.sh r02t 57
grep -E "dram__bytes|L2 Hit|Duration|Eligible|Issue|conflicts" gpurun_out/ncu_r02t_x57.txt
python scripts/sass_hot.py gpurun_out/src_r02t_x57.csv 5 3 | head -40

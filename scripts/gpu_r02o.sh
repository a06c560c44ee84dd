set -u
mkdir -p gpurun_out
DETAIL_JSON=gpurun_out/detail_c4d4_r02o.json timeout 300 python scripts/bench_detail.py c4d4 > /dev/null 2>&1
python scripts/show_detail.py gpurun_out/detail_c4d4_r02o.json 4
WL=c4d4 KREGEX=bk_stream PROF_VARIANT=2 GBE_KERNEL_POLICY=stream bash scripts/gpu_prof.sh r02o 0
grep -E "dram__bytes|L2 Hit|Duration|Eligible|Issue" gpurun_out/ncu_r02o_x0.txt

# usage: bash tools/gpu_prof_final.sh — the round's evidence: bench (+ reference arm), all configs,
# ncu launch lists with DRAM bytes (c2, c3, c5; host-driven loop: the graph's kernels), ncu --set full
# of the int32 and f64 8-way count + scatter (level 0) and the largest int32 leaf
cd $GRAFT_REPO_ROOT
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo BENCH $?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo REF $?
python tools/time_configs.py > gpurun_out/cfg_final.jsonl 2>&1; echo CFG $?
export BQ_HOST_LOOP=1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_c2_final.csv python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/n_c2.log 2>&1; echo NCU_C2 $?
for c in c3 c5; do
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_${c}_final.csv python tools/one_sort.py $c > gpurun_out/n_$c.log 2>&1; echo NCU_$c $?
done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_mw8t_scatter|k_mw8w_count' -s 0 -c 2 -o gpurun_out/final_mw8i python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/n7.log 2>&1; echo MW8I $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_leaf.*KI32.*512' -s 1 -c 1 -o gpurun_out/final_leaf python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/n8.log 2>&1; echo LEAF $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_mw8t_scatter|k_mw8w_count' -s 0 -c 2 -o gpurun_out/final_mw8w python tools/one_sort.py c3 > gpurun_out/n9.log 2>&1; echo MW8W $?

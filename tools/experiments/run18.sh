cp paper_2208_09822_b200/tuning/b200.tsv gpurun_out/b200_t18.tsv
for c in 5 1 4 3; do timeout 1500 python -m paper_2208_09822_b200.tune --config $c --out gpurun_out/b200_t18.tsv --log gpurun_out/tune18_c$c.log > /dev/null 2>&1; echo tune$c=$?; done

O=gpurun_out/prof_big; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hvp_reg_kernel -c 1 -s 2 -o $O/rb32 -f python tools/prof_one.py rosenbrock 32 16 hvp 262144 > $O/rb32.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:hvp_reg_kernel -c 1 -s 2 -o $O/rb64 -f python tools/prof_one.py rosenbrock 64 16 hvp 65536 > $O/rb64.log 2>&1
for k in rb32 rb64; do ncu -i $O/$k.ncu-rep --page details > $O/${k}_details.txt 2>&1; ncu -i $O/$k.ncu-rep --page raw --csv > $O/${k}_raw.csv 2>&1; ncu -i $O/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_source.csv 2>&1; done
ls -la $O

#!/bin/bash
# ncu executed-FLOP entries for the F3 rows of the DESIGN §10 table that had none
set -x
O=gpurun_out/r02f3g; mkdir -p $O
cp profiles/executed_flops.json gpurun_out/executed_flops.json
X="bash tools/ncu_executed.sh"
$X f3n4 --n 4 --m 1048576 --funcs fletcher_powell --csizes 4 > $O/ncu_f3n4.txt 2>&1
$X f3n8 --n 8 --m 1048576 --funcs fletcher_powell --csizes 8 > $O/ncu_f3n8.txt 2>&1
$X f3n32 --n 32 --m 65536 --funcs fletcher_powell --csizes 32 > $O/ncu_f3n32.txt 2>&1
$X f3n64sym --n 64 --m 16384 --funcs fletcher_powell --csizes 8 --algo sym_hvp > $O/ncu_f3n64sym.txt 2>&1
cp gpurun_out/executed_flops.json $O/
mv gpurun_out/sweep_* $O/ 2>/dev/null
cat $O/ncu_*.txt | grep -v "^=="

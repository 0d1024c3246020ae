#!/bin/bash
o=gpurun_out/proto4; mkdir -p $o
cd tools
./panel_proto 4800000 1800000 1800000 100000000 18 18 1 > ../$o/check.txt 2>&1
./panel_proto 4800000 1800000 1800000 1700000000 18 18 > ../$o/m0_18_18.txt 2>&1
./panel_proto 4800000 1800000 1800000 1700000000 17 17 > ../$o/m0_17_17.txt 2>&1
./panel_proto 1800000 4800000 1800000 1700000000 18 18 > ../$o/m1_18_18.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pipe2_kernel -s 1 -c 1 -o ../$o/ncu_pipe2 ./panel_proto 4800000 1800000 1800000 1700000000 18 18 0 2 > ../$o/ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pipe2_kernel -s 1 -c 1 -o ../$o/ncu_pipe2_fake ./panel_proto 4800000 1800000 1800000 1700000000 18 18 0 4 > ../$o/ncu2.log 2>&1

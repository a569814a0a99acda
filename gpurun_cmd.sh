timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r1_final.json 2> gpurun_out/bench_r1_final.err; echo "bench rc=$?"
for M in resnet18 resnet50 vit_b16; do
timeout 900 ncu --profile-from-start off --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/${M}_traffic.csv python tools/step_traffic.py $M gpurun_out/${M}_ops.json > gpurun_out/${M}_traffic.log 2>&1
echo "$M traffic rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_resnet18_bench.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
mkdir -p /tmp/nc
CDP_ARCH=resnet18 ONLY=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemm_pk_kernel<.int.0, .int.64, .bool.0, .bool.1, cdp::EpiConvOut2<.int.0>, .int.1" --launch-count 1 -o /tmp/nc/rn18_fprop64_full python tools/resnet_probe.py > /dev/null 2>&1
CDP_ARCH=resnet18 ONLY=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:gemm_pk_kernel<.int.0, .int.64, .bool.1, .bool.1, cdp::EpiHop2" --launch-count 1 -o /tmp/nc/rn18_wgrad64_full python tools/resnet_probe.py > /dev/null 2>&1
for f in fprop64 wgrad64; do
python tools/ncu_summary.py /tmp/nc/rn18_${f}_full.ncu-rep > gpurun_out/rn18_${f}_summary.json
ncu -i /tmp/nc/rn18_${f}_full.ncu-rep --page details --csv > gpurun_out/rn18_${f}_details.csv 2>/dev/null
done
cp /tmp/nc/rn18_fprop64_full.ncu-rep gpurun_out/

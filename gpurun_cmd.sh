for M in resnet18 resnet50 vit_b16; do
timeout 900 ncu --profile-from-start off --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file gpurun_out/${M}_traffic.csv python tools/step_traffic.py $M gpurun_out/${M}_ops.json > gpurun_out/${M}_traffic.log 2>&1
echo "$M rc=$?"; tail -2 gpurun_out/${M}_traffic.log
done

mkdir -p gpurun_out
for C in c2 c3; do
rm -f /tmp/nvlid_$C
PACT_LINK_TIMEOUT_MS=120000 timeout 400 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pack_lm|unpack|p2p_fold|p2p_gather" --csv --log-file gpurun_out/r2_nvlink_$C.csv python tools/nvlink_profile.py 0 2 /tmp/nvlid_$C $C > gpurun_out/r2_nvlink_${C}_r0.log 2>&1 &
P0=$!
PACT_LINK_TIMEOUT_MS=120000 timeout 400 python tools/nvlink_profile.py 1 2 /tmp/nvlid_$C $C > gpurun_out/r2_nvlink_${C}_r1.log 2>&1
wait $P0
tail -3 gpurun_out/r2_nvlink_${C}_r0.log
done

nproc; lscpu | grep -E "NUMA|Socket|Model name|^CPU\(s\)"; ls /sys/devices/system/node/ | grep node
B=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//; s/^0*//'); echo bus $B
for d in /sys/bus/pci/devices/*; do if [ -f $d/numa_node ]; then :; fi; done
P=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z'); P=${P#0000}; echo $P
cat /sys/bus/pci/devices/0000${P#0000}/numa_node 2>/dev/null || cat /sys/bus/pci/devices/$P/numa_node
cat /sys/bus/pci/devices/0000${P#0000}/local_cpulist 2>/dev/null
cat /proc/self/status | grep -i cpus_allowed_list
numactl --hardware 2>&1 | head -5
python scripts/exp_pcie.py 2>&1 | tail -5

set -x
nproc; lscpu | head -20; free -g; df -h; df -h /tmp /root /dev/shm; mount | grep -E " / | /tmp " ; nvidia-smi; nvidia-smi topo -m
cat /proc/meminfo | head -5
ulimit -a
dd if=/dev/zero of=/tmp/ddtest bs=1M count=8192 oflag=direct 2>&1 | tail -1
dd if=/tmp/ddtest of=/dev/null bs=1M iflag=direct 2>&1 | tail -1
rm -f /tmp/ddtest

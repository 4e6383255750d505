set -x
nproc; lscpu | head -20; free -g; df -h . /tmp /dev/shm; mount | grep -E " / | /tmp | /dev/shm" ; nvidia-smi; nvidia-smi topo -m
cat /proc/meminfo | head -5
ls /usr/local/cuda/lib64 | grep -i -E "cufile|nvcomp" 
dd if=/dev/zero of=./ddtest bs=1M count=4096 conv=fdatasync 2>&1 | tail -1
sync; echo 3 > /proc/sys/vm/drop_caches && echo dropped
dd if=./ddtest of=/dev/null bs=1M 2>&1 | tail -1
dd if=./ddtest of=/dev/null bs=1M 2>&1 | tail -1
rm -f ddtest
lsblk; cat /proc/mounts | head -30
python -c "import torch;print(torch.cuda.get_device_properties(0))"

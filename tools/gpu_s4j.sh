echo "default (4 GB / 16384)"; python tools/sp_time.py
echo "2 GB / 8192"; RLRA_B200_SWEEP_BYTES=2147483648 RLRA_B200_SWEEP_PANEL=8192 python tools/sp_time.py

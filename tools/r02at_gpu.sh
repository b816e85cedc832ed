N=131072 timeout 600 python tools/route_fa_sms.py 2>&1 | tail -3
N=32768 SMS=0,16,32,48,64,74,96 timeout 600 python tools/route_fa_sms.py 2>&1 | tail -3

timeout 300 python tools/order_test.py > gpurun_out/order.log 2>&1
sleep 20; KEEP=1 timeout 300 python tools/order_test.py >> gpurun_out/order.log 2>&1

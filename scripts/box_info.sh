# GPU box facts next to a timing: clocks, memory clock, ECC, power limit, driver
nvidia-smi --query-gpu=name,serial,pci.bus_id,driver_version,clocks.max.sm,clocks.max.mem,clocks.mem,ecc.mode.current,power.limit,temperature.gpu --format=csv

# pass-2 forms over the pixel count W (C3: 25 k jobs, C5: 335 k jobs)
for W in 1024 4096 16384; do python tools/pass2_probe.py C3 20 $W auto,list,jobs; done
for W in 1024 4096 16384 65536; do python tools/pass2_probe.py C5 15 $W auto,list,jobs; done
for W in 256 1024 4096; do python tools/pass2_probe.py C2 30 $W auto,inline,list,jobs; done

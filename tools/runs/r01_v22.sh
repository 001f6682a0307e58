for b in 0 1 0 1 0 1; do echo "balance=$b"; LLEP_ROUTER_BALANCE=$b python tools/router_bench.py g120; LLEP_ROUTER_BALANCE=$b python tools/router_bench.py q3; done 2>&1 | grep -v Warn | cut -c1-200

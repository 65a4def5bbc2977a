# r03f: column I/O skeleton with half the rows by per-thread LDG (A2) vs TMA only (A)
timeout 120 ./scripts/micro/tma_cluster

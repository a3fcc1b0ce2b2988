"""CPU oracle for the SP-MoE verification-time expert path — TEST
INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py cpu_baseline /
--impl reference).  The product package never imports this."""

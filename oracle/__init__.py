"""oracle -- TEST INFRASTRUCTURE ONLY: the CPU checkers of the PMP hot path
(a plain-C restatement of the reference engine and the reference itself
compiled from /root/reference).  Never imported by the product package."""

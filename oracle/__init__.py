# TEST INFRASTRUCTURE ONLY: the fp64 CPU oracle and the reference-pinning shim.

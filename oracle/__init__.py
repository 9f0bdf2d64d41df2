"""CPU oracle and compiled-reference access -- TEST INFRASTRUCTURE ONLY."""

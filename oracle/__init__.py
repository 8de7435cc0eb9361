"""TEST INFRASTRUCTURE ONLY: CPU checkers (restatement + compiled reference)."""

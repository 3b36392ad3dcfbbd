"""B200-native Symbiosis base executor."""
